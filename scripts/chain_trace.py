"""Backward-chain clock64 timeline (CRVPINN_CHAIN_TRACE) of cluster 0 on C5: one eager loss_grad.
usage: python scripts/chain_trace.py [C5] ; report: python scripts/chain_trace.py --report file
Needs a library built with the timeline macros: scripts/ab_build_tc.sh trace -DCRV_TRACE=1, then
CRVPINN_LIB=build/ab/trace/libcrvpinn.so (the default build compiles them out of the hot loops).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if sys.argv[1:2] == ["--report"]:
    t = np.fromfile(sys.argv[2], dtype=np.int64).reshape(8, 512)
    t0 = t[t > 0].min()
    names = ["p:tempty?", "p:tempty ok", "m:tfull ok", "m:issued", "e:wait x", "e:x ok", "e:done", "m:xempty ok"]
    for cta in range(8):
        r = t[cta]
        if (r <= 0).all():
            continue
        print(f"CTA {cta}:")
        for k in list(range(0, 6)) + list(range(60, 64)):
            ev = r[k * 8:(k + 1) * 8]
            print(f"  k={k:3d} " + " ".join(f"{names[e]}={int(ev[e] - t0) if ev[e] > 0 else -1:7d}" for e in range(8)))
        m = r[3::8]
        m = m[m > 0]
        if len(m) > 2:
            d = np.diff(m)
            print(f"  MMA issue-done period: median {np.median(d):.0f} cyc, mean {d.mean():.0f} over {len(d)} tiles")
    sys.exit(0)
sys.path.insert(0, ROOT)
import paper_2604_20731_b200 as crv  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
F = W.make_fields(name)
w = F.workload
g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=crv.PREC_TENSOR, lr=w.lr)
g.loss_grad()
os.environ["CRVPINN_CHAIN_TRACE"] = os.path.join(ROOT, "gpurun_out", "chain_trace.bin")
g.loss_grad()
print("ok")
