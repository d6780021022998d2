"""Throughput of crvpinn_eval_points (continuous evaluation) on the C5 network:
n = (512 x 3)^2 = 2,359,296 points (a 3x3 Gauss rule on the 512^2 IGA mesh), random in the unit square.
Reports the end-to-end C-ABI call from pageable host buffers (H2D of xy, kernels, D2H of p; wall
clock, mean of reps after one warm-up call), both precisions.
usage: python scripts/bench_eval_points.py [reps]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_20731_b200 as crv  # noqa: E402
import workloads as W  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
F = W.make_fields("C5")
w = F.workload
n = (512 * 3) ** 2
xy = np.random.default_rng(0).uniform(0, 1, (n, 2)).astype(np.float32)
wd = w.widths
flops_pt = 2 * (2 * wd[1] + sum(wd[l] * wd[l + 1] for l in range(1, len(wd) - 2)) + wd[-2])
out = {}
for prec, name in ((crv.PREC_TENSOR, "tensor"), (crv.PREC_FP32, "fp32")):
    g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=prec, lr=w.lr)
    g.eval_points(xy)
    t0 = time.perf_counter()
    for _ in range(reps):
        g.eval_points(xy)
    dt = (time.perf_counter() - t0) / reps
    out[name] = {"points": n, "e2e_ms": dt * 1e3, "e2e_points_per_s": n / dt,
                 "alg_tflops_e2e": n * flops_pt / dt / 1e12}
    g.close()
print(json.dumps({"op": "crvpinn_eval_points", "workload": "C5 network, 3x3 Gauss points of the 512^2 mesh",
                  "flops_per_point": flops_pt, **out}))
