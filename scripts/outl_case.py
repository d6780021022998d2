"""Debug helper: one loss_grad on a small tensor-path problem vs the oracle. usage: outl_case.py N w L"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import oracle  # noqa: E402
import paper_2604_20731_b200 as crv  # noqa: E402
import workloads as W  # noqa: E402

N, w, L = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
widths = (2,) + (w,) * L + (1,)
K, S, f = W.random_fields(N, 7)
th = W.random_theta(widths, 7)
g = crv.Crvpinn(N, widths, K, S, f, th, precision=crv.PREC_TENSOR)
loss, grad = g.loss_grad()
ref = oracle.Oracle(N, widths, K, S, f, th)
rl, rg = ref.loss_grad()
print(f"N={N} widths={widths}: loss {loss:.6e} ref {rl:.6e} rel {abs(loss - rl) / abs(rl):.2e} "
      f"grad rel-L2 {np.linalg.norm(grad - rg) / np.linalg.norm(rg):.2e}", flush=True)
for off, shape in W.theta_slices(widths):
    n = int(np.prod(shape))
    a, b = grad[off:off + n], rg[off:off + n]
    print(f"   {shape}: rel-L2 {np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30):.2e}  |ref| {np.linalg.norm(b):.3e}")
