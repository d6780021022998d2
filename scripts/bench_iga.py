"""f3 measurement: the IGA-ADS saturation step (crvpinn_iga_saturation_step) and the L2 projection on the
GPU at the paper's 100x100 quadratic-spline mesh and at 512x512, device time (CUDA events around the
kernels) and end to end from host buffers, next to the fp64 oracle (iga_oracle.c, 1 call).
usage: python scripts/bench_iga.py [reps]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_20731_b200 as crv  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
out = {"op": "crvpinn_iga_saturation_step / crvpinn_iga_project", "degree": 2}
for ne in (100, 512):
    g = crv.Iga(ne, 2)
    q = g.quad_points()
    rng = np.random.default_rng(ne)
    S = g.project(np.exp(-((q[:, 0] - 0.5) ** 2 + (q[:, 1] - 0.4) ** 2) / 0.02).astype(np.float32))
    S[0, :] = S[-1, :] = S[:, 0] = S[:, -1] = 0
    P = g.project((np.cos(2 * q[:, 0]) * q[:, 1]).astype(np.float32))
    K = np.exp(rng.standard_normal((ne, ne)) * 0.5).astype(np.float32)
    src = np.zeros((ne, ne), np.float32)
    src[ne // 3:ne // 2, ne // 3:ne // 2] = 1.0
    g.saturation_step(S, P, K, src, tau=0.01, gravity=1.0)
    dev, t0 = [], time.perf_counter()
    for _ in range(reps):
        g.saturation_step(S, P, K, src, tau=0.01, gravity=1.0)
        dev.append(g.last_ms)
    e2e = (time.perf_counter() - t0) / reps
    f = np.sin(3 * q[:, 0]).astype(np.float32)
    g.project(f)
    pdev = []
    for _ in range(reps):
        g.project(f)
        pdev.append(g.last_ms)
    e = {"n_elements": ne, "n_basis": g.nb, "quad_points": g.nq, "step_device_ms": float(np.median(dev)),
         "step_e2e_ms": e2e * 1e3, "project_device_ms": float(np.median(pdev))}
    import oracle
    o = oracle.IgaOracle(ne, 2)
    t0 = time.perf_counter()
    o.saturation_step(S.astype(np.float64), P.astype(np.float64), K.astype(np.float64), src.astype(np.float64),
                      tau=0.01, gravity=1.0)
    e["oracle_step_s"] = time.perf_counter() - t0
    out[f"ne{ne}"] = e
print(json.dumps(out))
