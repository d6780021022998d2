"""A/B numerics: the loss history of one step(100) on a workload, saved for comparison between builds.
usage: CRVPINN_LIB=... python scripts/bitcmp.py C4 out.npy"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_20731_b200 as crv
import workloads as W
F = W.make_fields(sys.argv[1]); w = F.workload
g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr)
h = g.step(100)
np.save(sys.argv[2], np.concatenate([h, g.theta.astype(np.float64)]))
