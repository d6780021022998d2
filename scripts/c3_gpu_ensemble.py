"""C3's schedule on the GPU -- pretraining (2000 Adam iterations) then 10 updates of 100 -- from theta0
and from ulp-perturbed copies (same perturbation recipe as scripts/c3_sensitivity.py), both precisions;
loss histories -> gpurun_out/c3_gpu_ensemble.npz. usage: python scripts/c3_gpu_ensemble.py [n_seeds]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_20731_b200 as m  # noqa: E402
import workloads as W  # noqa: E402

ns = int(sys.argv[1]) if len(sys.argv) > 1 else 8
F = W.make_fields("C3")
w = F.workload
out = {}
for prec in (1, 0):
    for seed in range(ns + 1):
        t0 = F.theta0.astype(np.float32)
        if seed > 0:
            rng = np.random.default_rng(seed)
            t0 = np.nextafter(t0, np.where(rng.random(t0.shape) < 0.5, -np.inf, np.inf).astype(np.float32))
        g = m.Crvpinn(w.N, w.widths, F.K, F.S, F.f, t0, precision=prec, lr=w.lr)
        out[f"p{prec}_s{seed}"] = np.concatenate([g.pretrain(2000)] + [g.step(100) for _ in range(10)])
        g.close()
np.savez(os.path.join(ROOT, "gpurun_out", "c3_gpu_ensemble.npz"), **out)
print("done")
