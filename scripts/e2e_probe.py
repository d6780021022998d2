"""Where the end-to-end step time goes (C5): device time of step(100) alone, with a device-resident
saturation update before it, and with a host one; host wall time of each call."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2604_20731_b200 as crv  # noqa: E402
import workloads as W  # noqa: E402

F = W.make_fields("C5")
w = F.workload
stream = torch.cuda.Stream()
g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr, stream=stream.cuda_stream)
S_dev = [torch.from_numpy(s).cuda() for s in F.S_steps]
for k in range(3):
    g.set_saturation(F.S_steps[k % len(F.S_steps)])
    g.step(100)
for mode in ("step", "device_S", "host_S", "host_S_hist"):
    td, th = [], []
    for k in range(6):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        if mode == "device_S":
            g.set_saturation_device(S_dev[k % len(S_dev)].data_ptr())
        elif mode.startswith("host_S"):
            g.set_saturation(F.S_steps[k % len(F.S_steps)])
        g.step(100, history=mode == "host_S_hist")
        e1.record(stream)
        torch.cuda.synchronize()
        th.append(time.perf_counter() - t0)
        td.append(e0.elapsed_time(e1))
    print(f"{mode:12s} device {np.median(td):.3f} ms  host wall {np.median(th)*1e3:.3f} ms")
