"""Write oracle-computed fixtures for the expensive parity cases (tests/golden/<cfg>_*.npz).

Calls only oracle/ and the seeded input generators (workloads/); nothing here touches the
CUDA path. Usage: python scripts/make_golden.py C3 C4 C5 [--steps 100]
Stored per config:
  theta0 fixture  <cfg>_theta0.npz : loss0 (fp64), grad0, u0, res0, q0, gu0 (float32)
  trajectory      <cfg>_traj<k>.npz: hist (fp64, k losses before each update), final_loss
                                     (LOSS(theta_k), fp64), theta_k (float32)
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def theta0_fixture(name):
    F = W.make_fields(name)
    w = F.workload
    t = time.time()
    o = oracle.Oracle(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr)
    loss, g, it = o.loss_grad(intermediates=True)
    np.savez_compressed(os.path.join(OUT, f"{name}_theta0.npz"), loss0=np.float64(loss),
                        grad0=g.astype(np.float32), u0=it["u"].astype(np.float32),
                        res0=it["res"].astype(np.float32), q0=it["q"].astype(np.float32),
                        gu0=it["gu"].astype(np.float32), threads=oracle.max_threads())
    print(f"{name} theta0: loss {loss:.9e}  {time.time() - t:.1f}s", flush=True)
    return o


def trajectory(name, steps, o=None):
    F = W.make_fields(name)
    w = F.workload
    t = time.time()
    if o is None:
        o = oracle.Oracle(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr)
    hist = o.train(steps)
    final = o.loss_grad()[0]
    np.savez_compressed(os.path.join(OUT, f"{name}_traj{steps}.npz"), hist=hist, final_loss=np.float64(final),
                        theta=o.theta.astype(np.float32), threads=oracle.max_threads())
    print(f"{name} traj{steps}: {hist[0]:.6e} -> {hist[-1]:.6e}, final {final:.6e}  {time.time() - t:.1f}s",
          flush=True)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    steps = 100
    if "--steps" in sys.argv:
        steps = int(sys.argv[sys.argv.index("--steps") + 1])
        args = [a for a in args if a != str(steps)]
    only_theta0 = "--theta0-only" in sys.argv
    for name in args:
        o = theta0_fixture(name)
        if not only_theta0:
            trajectory(name, steps, o)
