"""Run C3 pretraining (2000 Adam iterations) on the GPU in both precisions and save the loss
histories to gpurun_out/c3_pretrain_hist.npz (compared against tests/golden/C3_traj2000.npz)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_20731_b200 as m  # noqa: E402
import workloads as W  # noqa: E402

F = W.make_fields("C3")
w = F.workload
out = {}
for prec in (1, 0):
    g = m.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=prec, lr=w.lr)
    out[f"hist{prec}"] = g.pretrain(2000)
    out[f"final{prec}"] = g.loss_grad(grad=False)
    out[f"theta{prec}"] = g.theta
np.savez(os.path.join("gpurun_out", "c3_pretrain_hist.npz"), **out)
print("done")
