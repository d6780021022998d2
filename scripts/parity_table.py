"""Parity numbers of the five workloads for BASELINE.md: loss relative error and the largest per-tensor
gradient rel-L2 at theta0, and the relative difference of the final loss after 100 Adam steps, both
precisions, against the oracle (C1, C2 computed here; C3-C5 from tests/golden/, written by oracle/ only).
usage: python scripts/parity_table.py > gpurun_out/parity_table.json"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2604_20731_b200 as crv  # noqa: E402
import workloads as W  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def grad_err(widths, g, ref):
    gn = np.linalg.norm(ref)
    out = []
    for off, shape in W.theta_slices(widths):
        n = int(np.prod(shape))
        a, b = g[off:off + n].astype(np.float64), ref[off:off + n].astype(np.float64)
        out.append(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-3 * gn))
    return float(max(out))


res = {}
for name in W.WORKLOADS:
    F = W.make_fields(name)
    w = F.workload
    if name in ("C1", "C2"):
        o = oracle.Oracle(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr)
        rl, rg = o.loss_grad()
        o.train(100)
        rfinal = o.loss_grad()[0]
    else:
        z0 = np.load(os.path.join(GOLDEN, f"{name}_theta0.npz"))
        z1 = np.load(os.path.join(GOLDEN, f"{name}_traj100.npz"))
        rl, rg, rfinal = float(z0["loss0"]), z0["grad0"], float(z1["final_loss"])
    row = {}
    for prec, tag in ((crv.PREC_TENSOR, "tensor"), (crv.PREC_FP32, "fp32")):
        g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=prec, lr=w.lr)
        loss, grad = g.loss_grad()
        g.step(100, history=False)
        final = g.loss_grad(grad=False)
        g.close()
        row[tag] = {"loss_rel": abs(loss - rl) / abs(rl), "grad_rel_l2_max": grad_err(w.widths, grad, rg),
                    "final_loss_rel_100": abs(final - rfinal) / abs(rfinal)}
    res[name] = row
    print(name, json.dumps(row), file=sys.stderr, flush=True)
print(json.dumps(res))
