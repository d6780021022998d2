"""bench.py -- CRVPINN pressure-update throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5] [--precision tensor|fp32]
                    [--impl ours|reference] [--no-cpu-baseline]

A "step" is one pressure update of the paper (§6 step 7): the saturation
field is set (step A0) and 100 Adam iterations (A1..A8) run as one CUDA graph. The metric is
Adam iterations per second on the named workload (default C5, 512^2 grid, MLP 2-256x5-1).
value = Adam iterations of all ranks / max-over-ranks device time of the K timed steps,
inputs resident in HBM (device-side S). e2e = the same metric through the C ABI with host
buffers (H2D of S and D2H of the 100-entry loss history inside every step).
Multi-GPU: by default each rank runs an independent problem (replicas, scaling
"weak"); --shard splits ONE problem's MLP points over the ranks with two
in-graph NCCL all-reduces per Adam iteration (u after the forward, the gradient after the
backward), scaling "strong".
--impl reference times the fp64 CPU oracle (the reference arm of this tier) on the same config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

ITERS_PER_STEP = 100
# DRAM bytes per Adam iteration of the MLP kernels (forward + 4 backward GEMMs + weight-gradient
# reductions), ncu --set full at C5: profiles/r01_v8_ncu_full_summary.md (2.19e9 in v6-v8)
MLP_DRAM_BYTES_PER_ITER = 2.19e9


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--precision", default="tensor", choices=["tensor", "fp32"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--shard", action="store_true",
                    help="one problem, MLP points split over the ranks (strong scaling, NCCL exchanges)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ clocks during the timed region
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._proc = None

    def start(self):
        try:
            self._proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                           "--format=csv,noheader,nounits", "-lms", "200"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self._proc = None

    def _read(self):
        for line in self._proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) > 8:
                for k, nm in enumerate(names):
                    if r[5 + k].lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            return json.load(fh), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def alg_flops_per_iter(w: W.Workload) -> float:
    """forward + backward-dX + backward-dW flops per point x (N-1)^2 points."""
    ws = w.widths
    L = len(ws) - 2
    hid = ws[1]
    fwd = 2 * (2 * hid + (L - 1) * hid * hid + hid)
    bdx = 2 * ((L - 1) * hid * hid + hid)
    bdw = 2 * (2 * hid + (L - 1) * hid * hid + hid)
    return float(fwd + bdx + bdw) * w.points


def alg_bytes_per_iter(w: W.Workload) -> float:
    """alpha, b, u, RES/q, dLOSS/du through HBM once each (40 B/point) + 36 B/param."""
    return 40.0 * w.points + 36.0 * w.n_params


def measure_tf32_peak(device: int) -> float:
    """TF32 dense tensor peak of this GPU in TFLOP/s (torch.matmul 8192^3, TF32, best of 10)."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        a = torch.randn(8192, 8192, device=f"cuda:{device}")
        b = torch.randn(8192, 8192, device=f"cuda:{device}")
        best = float("inf")
        for _ in range(12):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        del a, b
        return 2.0 * 8192 ** 3 / best / 1e12
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


# ------------------------------------------------------------------ the oracle (CPU) arm
def time_oracle(name: str, iters: int):
    import oracle
    F = W.make_fields(name)
    w = F.workload
    t0 = time.perf_counter()
    o = oracle.Oracle(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr)
    t_factor = time.perf_counter() - t0
    t0 = time.perf_counter()
    o.train(iters)
    dt = time.perf_counter() - t0
    return iters / dt, oracle.max_threads(), t_factor


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    w = W.WORKLOADS[args.workload]
    import oracle
    F = W.make_fields(args.workload)
    t0 = time.perf_counter()
    o = oracle.Oracle(w.N, w.widths, F.K, F.S, F.f, F.theta0, lr=w.lr)
    t_factor = time.perf_counter() - t0
    # a step of the reference arm = 1 Adam iteration of the full workload (bounded sample)
    for _ in range(args.warmup):
        o.train(1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        o.train(1)
    dt = time.perf_counter() - t0
    value = args.steps / dt
    sample = (f"{args.steps} full Adam iterations of {args.workload} (1 per step) after {args.warmup} warm-up; "
              f"one-time banded-LU factorisation of G ({t_factor:.1f}s) excluded")
    line = {
        "impl": "reference", "metric": f"CRVPINN Adam iters/s ({args.workload})", "value": value,
        "unit": "Adam iters/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(workload_config(args.workload, "oracle"), adam_iters_per_step=1),
        "cpu_baseline": {"value": value, "unit": "Adam iters/s", "cores": oracle.max_threads(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "Adam iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(name: str, precision: str):
    w = W.WORKLOADS[name]
    return {"workload": f"{name}: {w.description}", "N": w.N, "grid": f"{w.N}x{w.N}",
            "points": w.points, "widths": list(w.widths), "params": w.n_params,
            "adam_iters_per_step": ITERS_PER_STEP, "lr": w.lr, "precision": precision,
            "l2": "flushed between timed steps (512 MiB device write, outside the per-step events)"}


# ------------------------------------------------------------------ our arm
def run_ours(args, rank, world, local):
    import torch
    import paper_2604_20731_b200 as crv

    # plumbing test hook: CRVPINN_BENCH_BACKEND=gloo lets several ranks share one GPU (functional check
    # of the multi-rank path only; such a run is not a measurement)
    backend = os.environ.get("CRVPINN_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    prec = crv.PREC_TENSOR if args.precision == "tensor" else crv.PREC_FP32
    F = W.make_fields(args.workload)
    w = F.workload
    stream = torch.cuda.Stream(device=torch.device("cuda", local))
    shard_kw, tile_frac = {}, 1.0
    if args.shard:
        nid = crv.share_nccl_id() if dist else crv.nccl_unique_id()
        shard_kw = dict(shard=(rank, world), nccl_id=nid)
        tile_frac = crv.shard_tiles(w.N, rank, world)[1] / (w.N * w.N // 128)
    g = crv.Crvpinn(w.N, w.widths, F.K, F.S, F.f, F.theta0, precision=prec, lr=w.lr, device=local,
                    stream=stream.cuda_stream, **shard_kw)
    S_dev = [torch.from_numpy(s).to(f"cuda:{local}") for s in F.S_steps]
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    torch.cuda.synchronize()

    def one_step(k):
        g.set_saturation_device(S_dev[k % len(S_dev)].data_ptr())
        g.step(ITERS_PER_STEP, history=False)

    for k in range(args.warmup):
        one_step(k)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    evs = []
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(float(k))            # L2 flush (outside the timed events)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        one_step(k)
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    sampler.stop()
    t_ms = sum(a.elapsed_time(b) for a, b in evs)
    # per-stage device times (roofline "achieved"): the same graph with CUDA event nodes between the
    # stages (cudaEventRecordExternal on the library stream), run right after the timed region --
    # the event nodes are kept out of the timed graph because they break kernel-to-kernel overlap
    g.set_profiling(True)
    one_step(0)                      # capture the profiled graph
    g.profile(reset=True)
    for k in range(max(2, min(args.steps, 5))):
        one_step(k)
    torch.cuda.synchronize()
    stage_ms, prof_iters = g.profile(reset=True)
    g.set_profiling(False)
    red_dev = f"cuda:{local}" if backend == "nccl" else "cpu"   # where the max-over-ranks reductions run
    t = torch.tensor([t_ms], dtype=torch.float64, device=red_dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    iters_total = (1 if args.shard else world) * args.steps * ITERS_PER_STEP
    value = iters_total / (t_max / 1e3)

    # e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        hist_bytes = ITERS_PER_STEP * 8
        s_bytes = F.S_steps[0].nbytes
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for k in range(args.steps):
            g.set_saturation(F.S_steps[k % len(F.S_steps)])
            g.step(ITERS_PER_STEP, history=True)
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], dtype=torch.float64, device=red_dev)
        if dist:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": iters_total / float(tt.item()), "unit": "Adam iters/s",
               "h2d_bytes_per_step": s_bytes, "d2h_bytes_per_step": hist_bytes}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return 0

    peaks, peak_src = measured_peaks()
    flops = alg_flops_per_iter(w) * tile_frac     # this rank's share of the MLP points
    mlp_ms = (stage_ms[0] + stage_ms[2]) / max(prof_iters, 1)
    achieved_tf = flops / (mlp_ms * 1e-3) / 1e12
    if prec == crv.PREC_TENSOR:
        # fp16 operands run at the bf16 rate; the MLP is timed inside a long step -> sustained
        peak = float(peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]))
        bound, peak_note = "tensor", f"{peak_src} bf16 sustained (fp16 = bf16 rate)"
    else:
        peak = 148 * 128 * 2 * 1.965e9 / 1e12   # FFMA fp32: SMs x lanes x 2 x max clock
        bound, peak_note = "alu", "derived FP32 FFMA peak 74.4 TFLOP/s (148 SM x 128 x 2 x 1965 MHz)"
    clocks = sampler.summary()
    # north_star / SURVEY.md §8(d) roofline: the method's precision class is TF32 (the fp16 operands
    # here have TF32's 10-bit mantissa), so its denominator is the TF32 tensor peak -- measured here
    # like MEASURED_PEAKS measures bf16 (torch.matmul 8192^3, TF32 enabled, best of 10) -- and the
    # whole Adam iteration is compared with max(GEMM flops / TF32 peak, algorithmic bytes / HBM).
    tf32 = measure_tf32_peak(local) if prec == crv.PREC_TENSOR else None
    step_s = (t_max / 1e3) / (args.steps * ITERS_PER_STEP)
    alg_bytes = alg_bytes_per_iter(w)
    line_ns = None
    if tf32:
        t_roof = max(flops / (tf32 * 1e12), alg_bytes / (float(peaks["hbm_gbs"]) * 1e9))
        line_ns = {"denominator": "TF32 tensor peak measured in this run (torch.matmul 8192^3, best of 10)",
                   "tf32_tflops": tf32, "t_roof_us": t_roof * 1e6, "step_us": step_s * 1e6,
                   "frac": t_roof / step_s}
    line = {
        "metric": f"CRVPINN Adam iters/s ({args.workload})", "value": value, "unit": "Adam iters/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.shard else "weak", "vs_baseline": None,
        "dtype": "f16" if prec == crv.PREC_TENSOR else "f32", "data": "synthetic",
        "config": dict(workload_config(args.workload, args.precision), parallelism=f"points{world}" if args.shard else f"replicas{world}"),
        "points_iters_per_s": value * w.points,
        "roofline": {"bound": bound, "achieved": achieved_tf, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved_tf / peak,
                     "traffic": MLP_DRAM_BYTES_PER_ITER if args.workload == "C5" and not args.shard else None,
                     "kernel": "MLP forward + backward (A1, A6-A7), per Adam iteration",
                     "alg_flops_per_iter": flops, "peak_source": peak_note,
                     "traffic_note": ("per-iteration DRAM bytes (read + write) of the MLP kernels from one ncu --set full "
                                     "capture at C5 (profiles/r01_v8_ncu_full_summary.md): the fp16 activations pass "
                                     "through HBM, so traffic >> the 20 MB algorithmic bytes; measured at C5 only")},
        "north_star_roofline": line_ns,
        "stage_ms_per_iter": {"mlp_fwd": stage_ms[0] / max(prof_iters, 1),
                              "stencil_gram_loss_adjoint": stage_ms[1] / max(prof_iters, 1),
                              "mlp_bwd_reduce": stage_ms[2] / max(prof_iters, 1),
                              "adam": stage_ms[3] / max(prof_iters, 1)},
        "clocks": clocks,
        "e2e": e2e,
        "gpu_launches": args.steps * (ITERS_PER_STEP * g.launches_per_iter + 1),
    }
    if world == 1 and not args.no_cpu_baseline:
        v, cores, t_factor = time_oracle(args.workload, 1)
        line["cpu_baseline"] = {"value": v, "unit": "Adam iters/s", "cores": cores, "kind": "oracle",
                                "sample": f"1 full Adam iteration of {args.workload} (fp64 oracle, OpenMP); "
                                          f"one-time LU factorisation ({t_factor:.1f}s) excluded"}
    print(json.dumps(line), flush=True)
    g.close()
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
