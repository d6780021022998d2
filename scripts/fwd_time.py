"""Time the MLP forward alone (crvpinn_eval = forward + D2H of u) on a workload: wall-clock
mean over n calls after warm-up. Used for A/B builds via CRVPINN_LIB. usage: fwd_time.py [C5] [n]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import paper_2604_20731_b200 as crv  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50
F = W.make_fields(name)
w = F.workload
g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=crv.PREC_TENSOR, lr=w.lr)
for _ in range(5):
    g.eval()
t0 = time.perf_counter()
for _ in range(n):
    p = g.eval()
dt = (time.perf_counter() - t0) / n
print(f"{os.environ.get('CRVPINN_LIB', 'default')}: eval {dt * 1e3:.3f} ms  (u finite: {np.isfinite(p).all()})")
