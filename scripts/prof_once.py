"""Profiling driver: build a workload context and run eager loss_grad evaluations (no graph),
so ncu can pick individual kernels: python scripts/prof_once.py [C5] [n_evals]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2604_20731_b200 as crv  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
F = W.make_fields(name)
w = F.workload
g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=crv.PREC_TENSOR, lr=w.lr)
for _ in range(n):
    loss, _ = g.loss_grad()
print("loss", loss)
