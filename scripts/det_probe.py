"""Run-to-run determinism probe: the same loss_grad (and intermediates) K times in one process and in
fresh contexts; prints which outputs differ bitwise. usage: python scripts/det_probe.py C5 [K]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_20731_b200 as crv
import workloads as W
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
F = W.make_fields(name); w = F.workload
outs = []
for rep in range(K):
    g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr)
    for it in range(2):
        loss, grad = g.loss_grad()
        im = g.intermediates()
        outs.append((rep, it, loss, grad.copy(), im["u"].copy(), im["q"].copy(), im["gu"].copy()))
    h = g.step(20)
    outs.append((rep, 9, float(h[-1]), g.theta.copy(), h.copy(), None, None))
    g.close()
ref = {}
for rep, it, loss, a, b, c, d in outs:
    key = it
    if key not in ref:
        ref[key] = (loss, a, b, c, d)
        continue
    r = ref[key]
    same = [loss == r[0], np.array_equal(a, r[1]), np.array_equal(b, r[2]),
            (c is None) or np.array_equal(c, r[3]), (d is None) or np.array_equal(d, r[4])]
    extra = ""
    if not same[1]:
        extra = f" grad maxdiff {np.max(np.abs(a - r[1])):.3e} nnz {np.count_nonzero(a != r[1])}"
    print(f"{name} rep {rep} call {it}: loss/grad/u/q/gu equal {same}{extra}", flush=True)
