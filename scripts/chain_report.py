"""Per-stage breakdown of a backward-chain trace (slots per tile: 0/1 producer t wait, 2 MMA tfull,
3 MMA dX committed, 4/5 epilogue xfull wait, 6 epilogue done, 7 MMA xempty, 8 dX drained,
9 ring slot free, 10 math+stores done, 11-14 producer gfull waits (chunks 0, 1), 15 MMA chunk-0 data)."""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.int64).reshape(8, 64, 16)
med = lambda a, b, c: int(np.median(t[c, 5:60, b] - t[c, 5:60, a]))  # noqa: E731
for c in range(8):
    per = int(np.median(np.diff(t[c, 5:60, 3])))
    print(f"CTA {c}: period {per} | epi: xwait {med(4, 5, c)} tmem {med(5, 8, c)} oempty {med(8, 9, c)} "
          f"math {med(9, 10, c)} fence {med(10, 6, c)} | mma: tfull->chunk0 data {med(2, 15, c)} "
          f"dX issue {med(15, 3, c)} | prod gfull0 wait {med(11, 12, c)}")
