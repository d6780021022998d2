"""Two IGA-ADS saturation steps at ne = 512 (quadratic) for an ncu launch list."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_20731_b200 as crv  # noqa: E402

ne = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = crv.Iga(ne, 2)
q = g.quad_points()
S = g.project(np.exp(-((q[:, 0] - 0.5) ** 2 + (q[:, 1] - 0.4) ** 2) / 0.02).astype(np.float32))
P = g.project((np.cos(2 * q[:, 0]) * q[:, 1]).astype(np.float32))
K = np.ones((ne, ne), np.float32)
src = np.zeros((ne, ne), np.float32)
for _ in range(2):
    S2 = g.saturation_step(S, P, K, src, tau=0.01, gravity=1.0)
print(g.last_ms)
