"""Per-tile breakdown of a k_tc_bwd2 trace (CRVPINN_BWD_TRACE, CTA 0; slots per tile: 0/1 producer
t wait, 2 MMA tfull, 7 MMA xempty, 8-11 MMA chunk j data, 3 MMA done, 4/5 epilogue xfull wait,
6 epilogue done; output-layer launch: 12/13/14 Delta_L transform start, chunk 0 released, end).
usage: python scripts/bwd2_report.py file
Needs a library built with the timeline macros: scripts/ab_build_tc.sh trace -DCRV_TRACE=1, then
CRVPINN_LIB=build/ab/trace/libcrvpinn.so (the default build compiles them out of the hot loops).
"""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.int64)[:4096].reshape(256, 16)
n = int((t[:, 3] > 0).sum())
r = t[2:n - 2]
med = lambda a, b: int(np.median(r[:, b] - r[:, a]))  # noqa: E731
per = int(np.median(np.diff(r[:, 3])))
print(f"tiles {n}: period {per} | mma: tfull wait {int(np.median(r[:, 2] - t[1:n - 3, 3]))} xempty {med(2, 7)} "
      f"chunk0 {med(7, 8)} chunk1 {med(8, 9)} chunk2 {med(9, 10)} chunk3 {med(10, 11)} tail {med(11, 3)} | "
      f"epi: xwait {med(4, 5)} work {med(5, 6)}")
if (r[:, 12] > 0).all():   # output-layer launch: Delta_L transform (slots 12 start, 13 chunk 0 released, 14 end)
    print(f"outl transform: chunk0 {med(12, 13)} all {med(12, 14)} | transform end -> dX epilogue start "
          f"{med(14, 4)} | epilogue start -> next transform {int(np.median(t[3:n - 1, 12] - r[:, 6]))}")
