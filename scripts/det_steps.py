"""Run-to-run determinism of the graph step path: K fresh contexts each run step(n); prints whether each
rep's history and theta equal rep 0's bitwise. usage: python scripts/det_steps.py C5 [K] [n]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_20731_b200 as crv
import workloads as W
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 5
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
F = W.make_fields(name); w = F.workload
ref = None
res = []
for rep in range(K):
    g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr)
    h = g.step(n)
    th = g.theta.copy()
    g.close()
    import hashlib
    hh = hashlib.md5(h.tobytes() + th.tobytes()).hexdigest()[:8]
    print(f"{name} {os.environ.get('TAG', '')} rep {rep}: {hh} last loss {h[-1]:.10e}", flush=True)
    if ref is None:
        ref = (h, th)
        continue
    first = int(np.argmax(h != ref[0])) if not np.array_equal(h, ref[0]) else -1
    res.append(np.array_equal(h, ref[0]) and np.array_equal(th, ref[1]))
    print(f"{name} {os.environ.get('TAG', '')} rep {rep}: equal {res[-1]} first differing iteration {first}", flush=True)
print(f"{name} {os.environ.get('TAG', '')}: {sum(res)}/{len(res)} reps equal to rep 0")
