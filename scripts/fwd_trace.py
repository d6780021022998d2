"""clock64 timeline of the forward kernel's CTA 0 (debug build path, env CRVPINN_FWD_TRACE).
usage: python scripts/fwd_trace.py [C5] [out.bin] ; analysed by scripts/fwd_trace_report.py
Needs a library built with the timeline macros: scripts/ab_build_tc.sh trace -DCRV_TRACE=1, then
CRVPINN_LIB=build/ab/trace/libcrvpinn.so (the default build compiles them out of the hot loops).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "fwd_trace.bin")
import paper_2604_20731_b200 as crv  # noqa: E402
import workloads as W  # noqa: E402

F = W.make_fields(name)
w = F.workload
g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=crv.PREC_TENSOR, lr=w.lr)
g.eval()
os.environ["CRVPINN_FWD_TRACE"] = out
g.eval()
g.eval()
print("trace ->", out)
