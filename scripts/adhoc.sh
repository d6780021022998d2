#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "iga" > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
timeout -s KILL 600 python scripts/bench_iga.py > gpurun_out/iga.json 2>gpurun_out/iga.err; tail -c 900 gpurun_out/iga.json; tail -3 gpurun_out/iga.err
CRVPINN_IGA_ASSEMBLY=split timeout -s KILL 600 python scripts/bench_iga.py > gpurun_out/iga_split.json 2>&1; tail -c 900 gpurun_out/iga_split.json
python - <<'PY'
import sys, numpy as np, os
sys.path.insert(0, '.')
import paper_2604_20731_b200 as crv
# fused vs split assembly must agree bit for bit
res = {}
for mode in ("fused", "split"):
    if mode == "split": os.environ["CRVPINN_IGA_ASSEMBLY"] = "split"
    else: os.environ.pop("CRVPINN_IGA_ASSEMBLY", None)
    out = []
    for ne, r in ((37, 2), (20, 3), (24, 5), (512, 2)):
        g = crv.Iga(ne, r)
        q = g.quad_points()
        S = g.project(np.exp(-((q[:, 0] - 0.5) ** 2 + (q[:, 1] - 0.4) ** 2) / 0.02).astype(np.float32))
        P = g.project((np.cos(2 * q[:, 0]) * q[:, 1]).astype(np.float32))
        K = np.exp(np.random.default_rng(ne).standard_normal((ne, ne)) * 0.5).astype(np.float32)
        src = np.zeros((ne, ne), np.float32); src[ne // 3:ne // 2, ne // 3:ne // 2] = 1
        out.append((S, g.saturation_step(S, P, K, src, tau=0.01, gravity=1.0)))
    res[mode] = out
for (a1, b1), (a2, b2) in zip(res["fused"], res["split"]):
    print("rel diff", float(np.abs(b1 - b2).max() / np.abs(b2).max()))
PY
