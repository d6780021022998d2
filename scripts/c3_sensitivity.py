"""Sensitivity of C3 pretraining to rounding-level perturbations, oracle only (fp64).

Runs the oracle's 2000-iteration C3 pretraining from theta0 with every entry moved by one fp32 ulp
up or down (seeded signs; the oracle takes theta0 as fp32), and stores the loss history. Comparing it
with tests/golden/C3_traj2000.npz (unperturbed) measures how far two exact-arithmetic runs that
differ by fp32 rounding drift apart: the bound any fp32 / fp16 implementation can be held to.
usage: python scripts/c3_sensitivity.py [seed] [steps]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import workloads as W  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
F = W.make_fields("C3")
w = F.workload
rng = np.random.default_rng(seed)
t0 = F.theta0.astype(np.float32)
th = np.nextafter(t0, np.where(rng.random(t0.shape) < 0.5, -np.inf, np.inf).astype(np.float32))
t = time.time()
o = oracle.Oracle(w.N, w.widths, F.K, F.S, F.f, th, lr=w.lr)
hist = o.train(steps)
final = o.loss_grad()[0]
out = os.path.join(ROOT, "tests", "golden", f"C3_traj{steps}_perturbed{seed}.npz")
np.savez_compressed(out, hist=hist, final_loss=np.float64(final), seed=seed, threads=oracle.max_threads())
print(f"C3 perturbed seed {seed}: {hist[0]:.6e} -> {hist[-1]:.6e}, final {final:.6e}  {time.time() - t:.1f}s")
