import sys, os, numpy as np
sys.path.insert(0, '.')
import paper_2604_20731_b200 as crv, oracle
for ne, r in ((128, 2), (512, 2), (40, 3)):
    g = crv.Iga(ne, r)
    q = g.quad_points()
    S = g.project(np.exp(-((q[:, 0] - 0.5) ** 2 + (q[:, 1] - 0.4) ** 2) / 0.02).astype(np.float32))
    P = g.project((np.cos(2 * q[:, 0]) * q[:, 1]).astype(np.float32))
    K = np.exp(np.random.default_rng(ne).standard_normal((ne, ne)) * 0.5).astype(np.float32)
    src = np.zeros((ne, ne), np.float32); src[ne // 3:ne // 2, ne // 3:ne // 2] = 1
    o = oracle.IgaOracle(ne, r)
    ref = o.saturation_step(S.astype(np.float64), P.astype(np.float64), K.astype(np.float64), src.astype(np.float64), tau=0.01, gravity=1.0)
    for mode in ("fused", "split"):
        if mode == "split": os.environ["CRVPINN_IGA_ASSEMBLY"] = "split"
        else: os.environ.pop("CRVPINN_IGA_ASSEMBLY", None)
        out = g.saturation_step(S, P, K, src, tau=0.01, gravity=1.0)
        d = out - ref
        print(ne, r, mode, "max rel", float(np.abs(d).max() / np.abs(ref).max()), "rel l2", float(np.linalg.norm(d) / np.linalg.norm(ref)))
