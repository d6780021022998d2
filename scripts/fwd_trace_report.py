"""Summarise a forward clock64 trace (scripts/fwd_trace.py): per GEMM gi of CTA 0 the epilogue's
accumulator wait, chunk release times and the MMA issue times, in cycles relative to the first event.
usage: python scripts/fwd_trace_report.py gpurun_out/fwd_trace.bin [KC]"""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.int64)
KC = int(sys.argv[2]) if len(sys.argv) > 2 else 4
nz = t[t > 0]
t0 = nz.min()
rel = lambda v: (int(v - t0) if v > 0 else -1)  # noqa: E731
G = 0
while G * 16 + 5 < 2048 and (t[G * 16 + 2] > 0 or t[G * 16] > 0):
    G += 1
print("gi | acc_wait_start acc_ready | releases of A chunks (for GEMM gi) | MMA a_full / w_ready / issued per chunk")
prev = None
for gi in range(G):
    rs = [rel(t[gi * 16 + 2 + c]) for c in range(KC)]
    mm = [(rel(t[2048 + (gi * KC + c) * 4]), rel(t[2048 + (gi * KC + c) * 4 + 1]), rel(t[2048 + (gi * KC + c) * 4 + 2]))
          for c in range(KC)]
    aw = (rel(t[gi * 16]), rel(t[gi * 16 + 1]))
    d = [rs[c] - rs[c - 1] for c in range(1, KC)]
    print(f"{gi:3d} | {aw[0]:8d} {aw[1]:8d} | rel {rs} d={d} | mma {mm}")

# per-warp view (slots 1024..): for GEMM-epilogue gi < 12, acc-ready and chunk releases of the 16
# epilogue warps (warp w -> SMSP (w+2) % 4)
print("\nper-warp (rel. to warp 2's acc ready): gi: acc-ready spread | chunk c release min/max and slowest warps")
for gi in range(12):
    base = 1024 + gi * (KC + 1) * 16
    acc = t[base:base + 16]
    if (acc <= 0).all():
        continue
    ref = t[gi * 16 + 1]
    line = f"{gi:3d}: acc {int(acc.min() - ref):5d}..{int(acc.max() - ref):5d} |"
    for c in range(KC):
        r = t[base + (1 + c) * 16: base + (2 + c) * 16]
        order = np.argsort(r)
        line += f" c{c} {int(r.min() - ref):5d}..{int(r.max() - ref):5d} (slow w{order[-1] + 2},{order[-2] + 2})"
    print(line)
