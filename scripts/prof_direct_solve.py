"""One short direct solve at C5 (20 CG iterations) for an ncu launch list."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_20731_b200 as crv  # noqa: E402
import workloads as W  # noqa: E402

F = W.make_fields(sys.argv[1] if len(sys.argv) > 1 else "C5")
w = F.workload
g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0)
print(g.direct_solve(rtol=1e-12, max_iter=20)[1:])
