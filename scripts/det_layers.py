"""Localise a run-to-run difference of the step path: a reference context (CRVPINN_SIDE_REDUCE=0, no
side-stream reductions) and a default one run step(1) in lock step; after each call theta is compared
per parameter tensor and the first mismatch is reported. usage: python scripts/det_layers.py C5 [calls] [reps]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_20731_b200 as crv
import workloads as W
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 30
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
n_iter = int(os.environ.get("ITERS", "1"))
F = W.make_fields(name); w = F.workload
widths = w.widths
def tensors(th):
    out, o = [], 0
    for l in range(len(widths) - 1):
        nw, nb = widths[l] * widths[l + 1], widths[l + 1]
        out.append((f"W{l}", th[o:o + nw])); o += nw
        out.append((f"b{l}", th[o:o + nb])); o += nb
    return out
os.environ["CRVPINN_SIDE_REDUCE"] = "0"
ref = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr)
os.environ.pop("CRVPINN_SIDE_REDUCE")
href = [ref.step(n_iter) for _ in range(calls)]
thref = []
ref.close()
os.environ["CRVPINN_SIDE_REDUCE"] = "0"
ref = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr)
os.environ.pop("CRVPINN_SIDE_REDUCE")
for c in range(calls):
    ref.step(n_iter)
    thref.append(ref.theta.copy())
for rep in range(reps):
    g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr)
    for c in range(calls):
        h = g.step(n_iter)
        th = g.theta
        if not np.array_equal(th, thref[c]) or not np.array_equal(h, href[c]):
            diffs = [(nm, int(np.count_nonzero(a != b)), float(np.max(np.abs(a - b)))) for (nm, a), (_, b) in
                     zip(tensors(th), tensors(thref[c])) if not np.array_equal(a, b)]
            print(f"{name} rep {rep}: first mismatch after call {c} (hist equal {np.array_equal(h, href[c])}): {diffs}",
                  flush=True)
            break
    else:
        print(f"{name} rep {rep}: {calls} calls equal to the reference", flush=True)
    g.close()
