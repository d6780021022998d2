"""Per-stage device time per Adam iteration (profiled step graph: CUDA event nodes between the
stages) and the unprofiled step time, for A/B builds via CRVPINN_LIB.
usage: python scripts/stage_time.py [C5] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_20731_b200 as crv  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
F = W.make_fields(name)
w = F.workload
g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=crv.PREC_TENSOR, lr=w.lr)
g.step(100, history=False)
g.set_profiling(True)
g.step(100, history=False)
g.profile(reset=True)
for _ in range(reps):
    g.step(100, history=False)
st, n = g.profile(reset=True)
g.set_profiling(False)
g.step(100, history=False)
torch.cuda.synchronize()
stream = torch.cuda.ExternalStream(g.stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(reps):
    g.step(100, history=False)
e1.record(stream)
torch.cuda.synchronize()
it = e0.elapsed_time(e1) / (reps * 100)
lib = os.environ.get("CRVPINN_LIB", "default")
st = [x / max(n, 1) for x in st]
print(f"{lib}: fwd {st[0] * 1e3:.1f} fields {st[1] * 1e3:.1f} bwd {st[2] * 1e3:.1f} adam {st[3] * 1e3:.1f} us/iter"
      f" | step {it * 1e3:.1f} us/iter ({1e3 / it:.0f} it/s)")
