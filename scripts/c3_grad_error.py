"""Gradient error of the tensor path along C3's pretraining trajectory (reading R28).

The fp32 path trains C3 from theta0; at checkpoints its theta is loaded into a tensor-path
context and both gradients are taken at the same theta. Reports the tensor path's gradient error
(global and per-tensor rel-L2, cosine, and the projection coefficient <g_tc, g_32>/|g_32|^2, which
is 1 for an unbiased error) -> gpurun_out/c3_grad_error.npz (thetas included, so the oracle's
gradient at the same points can be computed on the CPU). usage: python scripts/c3_grad_error.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_20731_b200 as m  # noqa: E402
import workloads as W  # noqa: E402

F = W.make_fields("C3")
w = F.workload
f32 = m.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=m.PREC_FP32, lr=w.lr)
tc = m.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=m.PREC_TENSOR, lr=w.lr)
checks = [0, 100, 250, 500, 1000, 1500, 2000, 3000]
out = {"checks": np.array(checks)}
done = 0
for c in checks:
    if c > done:
        f32.step(c - done, history=False)
        done = c
    th = f32.theta
    tc.theta = th
    l32, g32 = f32.loss_grad()
    ltc, gtc = tc.loss_grad()
    g32 = g32.astype(np.float64)
    gtc = gtc.astype(np.float64)
    e = gtc - g32
    rel = np.linalg.norm(e) / np.linalg.norm(g32)
    cos = float(gtc @ g32 / (np.linalg.norm(gtc) * np.linalg.norm(g32)))
    proj = float(gtc @ g32 / (g32 @ g32))
    per = []
    for off, shape in W.theta_slices(w.widths):
        n = int(np.prod(shape))
        per.append(np.linalg.norm(e[off:off + n]) / max(np.linalg.norm(g32[off:off + n]), 1e-30))
    print(f"it {c:5d}: loss fp32 {l32:.6e} tensor {ltc:.6e} (rel {abs(ltc - l32) / l32:.2e})  grad rel-L2 {rel:.3e} "
          f"cos {cos:.8f} proj {proj:.6f}  per-tensor max {max(per):.3e}", flush=True)
    out[f"theta_{c}"] = th
    out[f"g32_{c}"] = g32.astype(np.float32)
    out[f"gtc_{c}"] = gtc.astype(np.float32)
    out[f"loss_{c}"] = np.array([l32, ltc])
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez_compressed(os.path.join(ROOT, "gpurun_out", "c3_grad_error.npz"), **out)
