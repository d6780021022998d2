"""Quick diagnostic: tensor-core (and fp32) path vs the oracle on small problems, printing the
error of every intermediate. Usage: python scripts/tc_check.py [prec] [cases...]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2604_20731_b200 as crv  # noqa: E402
import workloads as W  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def check(N, widths, seed, prec):
    K, S, f = W.random_fields(N, seed)
    th = W.random_theta(widths, seed)
    ref = oracle.Oracle(N, widths, K, S, f, th)
    rl, rg, it = ref.loss_grad(intermediates=True)
    t0 = time.time()
    g = crv.Crvpinn(N, widths, K, S, f, th, precision=prec)
    loss, grad = g.loss_grad()
    im = g.intermediates()
    print(f"N={N} widths={widths} prec={prec}  ({time.time() - t0:.2f}s)")
    print(f"   u rel {rel(im['u'], it['u']):.3e}  res rel {rel(im['res'], it['res']):.3e}  "
          f"q rel {rel(im['q'], it['q']):.3e}  gu rel {rel(im['gu'], it['gu']):.3e}")
    print(f"   loss {loss:.9e} vs {rl:.9e} rel {abs(loss - rl) / abs(rl):.3e}")
    for k, (off, shape) in enumerate(W.theta_slices(widths)):
        n = int(np.prod(shape))
        a, b = grad[off:off + n], rg[off:off + n]
        e = np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-3 * np.linalg.norm(rg))
        print(f"   grad[{k}] {shape}: rel-L2 {e:.3e}  |ref| {np.linalg.norm(b):.3e}")
    hist = g.step(5)
    rh = ref.train(5)
    print(f"   5 steps: {np.max(np.abs(hist - rh) / np.abs(rh)):.3e}")
    g.close()


if __name__ == "__main__":
    prec = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    cases = [(16, (2, 64, 64, 1), 0), (32, (2, 32, 32, 1), 1), (32, (2, 128, 128, 128, 1), 2),
             (16, (2, 256, 256, 1), 3), (64, (2, 256, 256, 256, 1), 4)]
    for N, widths, seed in cases:
        check(N, widths, seed, prec)
