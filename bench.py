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
    ap.add_argument("--no-per-workload", action="store_true", help="skip the C1-C5 table (per_workload)")
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
    sample = (f"{args.steps} full Adam iterations of {args.workload} (1 per step: a bounded sample of the 100-iteration "
              f"pressure update of the config) after {args.warmup} warm-up; "
              f"one-time banded-LU factorisation of G ({t_factor:.1f}s) excluded")
    line = {
        "impl": "reference", "metric": f"CRVPINN Adam iters/s ({args.workload})", "value": value,
        "unit": "Adam iters/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(workload_config(args.workload, args.precision), parallelism="replicas1"),
        "cpu_baseline": {"value": value, "unit": "Adam iters/s", "cores": oracle.max_threads(), "kind": "oracle",
                         "cpu": cpu_model(), "sample": sample},
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
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def set_oracle_threads(n: int) -> None:
    """OpenMP thread count of the oracle's parallel regions (libgomp ICV of this thread)."""
    import ctypes
    import oracle
    oracle.lib()
    ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(n))


# oracle Adam iterations timed per workload in the per-workload table (bounded samples)
ORACLE_ITERS = {"C1": 50, "C2": 10, "C3": 3, "C4": 1, "C5": 1}


def time_oracle_table(names, one_thread=("C1", "C2", "C3")):
    import oracle
    out = {}
    nmax = oracle.max_threads()
    for name in names:
        v, cores, _ = time_oracle(name, ORACLE_ITERS[name])
        row = {"value": v, "unit": "Adam iters/s", "cores": cores, "iters_timed": ORACLE_ITERS[name]}
        if name in one_thread:
            set_oracle_threads(1)
            try:
                row["value_1thread"] = time_oracle(name, ORACLE_ITERS[name])[0]
            finally:
                set_oracle_threads(nmax)
        out[name] = row
    return out


def roofline_frac(w, ms_per_iter, peak_tf):
    ach = alg_flops_per_iter(w) / (ms_per_iter * 1e-3) / 1e12
    return ach, ach / peak_tf


def measured_traffic():
    """Per-iteration DRAM bytes of the whole Adam iteration per workload, from one ncu --set full capture
    (profiles/r02_traffic.json, written by scripts/ncu_traffic.py); None where not captured."""
    path = os.path.join(ROOT, "profiles", "r02_traffic.json")
    if not os.path.exists(path):
        return {}, None
    with open(path) as fh:
        d = json.load(fh)
    return d.get("bytes_per_iter", {}), d.get("source")


def time_steps(torch, g, S_dev, stream, flush, steps, warmup):
    """Device time (ms) of `steps` pressure updates (set_saturation + 100-iteration graph), L2 flushed
    between them outside the events."""
    def one_step(k):
        g.set_saturation_device(S_dev[k % len(S_dev)].data_ptr())
        g.step(ITERS_PER_STEP, history=False)
    for k in range(warmup):
        one_step(k)
    torch.cuda.synchronize()
    evs = []
    for k in range(steps):
        with torch.cuda.stream(stream):
            flush.fill_(float(k))
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        one_step(k)
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs), one_step


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

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t_ms, one_step = time_steps(torch, g, S_dev, stream, flush, args.steps, args.warmup)
    if dist:
        dist.barrier()
    sampler.stop()
    # per-stage device times (the dominant kernel's share): the same graph with CUDA event nodes between
    # the stages (cudaEventRecordExternal on the library stream), run right after the timed region --
    # the event nodes are kept out of the timed graph because they break kernel-to-kernel overlap
    g.set_profiling(True)
    one_step(0)                      # capture the profiled graph
    g.profile(reset=True)
    for k in range(max(2, min(args.steps, 5))):
        one_step(k)
    torch.cuda.synchronize()
    stage_ms, prof_iters = g.profile(reset=True)
    g.set_profiling(False)
    # leaving profiling mode drops the captured graphs: re-capture the step graph here (one untimed
    # step) so that the end-to-end loop below times steady-state steps, not a graph instantiation
    g.step(ITERS_PER_STEP, history=True)
    torch.cuda.synchronize()
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
    launches = args.steps * (ITERS_PER_STEP * g.launches_per_iter + 1)

    if rank != 0:
        g.close()
        if dist:
            dist.destroy_process_group()
        return 0

    peaks, peak_src = measured_peaks()
    traffic, traffic_src = measured_traffic()
    flops = alg_flops_per_iter(w) * tile_frac     # this rank's share of the MLP points
    ms_iter = t_max / (args.steps * ITERS_PER_STEP)
    if prec == crv.PREC_TENSOR:
        # fp16 operands run at the bf16 rate; every kernel runs inside a long step -> the sustained figure
        peak = float(peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]))
        bound, peak_note = "tensor", f"{peak_src} bf16 sustained (fp16 = bf16 rate), MEASURED_PEAKS.json"
    else:
        peak = 148 * 128 * 2 * 1.965e9 / 1e12   # FFMA fp32: SMs x lanes x 2 x max clock
        bound, peak_note = "alu", "derived FP32 FFMA peak 74.4 TFLOP/s (148 SM x 128 x 2 x 1965 MHz)"
    achieved = flops / (ms_iter * 1e-3) / 1e12
    pi = max(prof_iters, 1)
    st = {"mlp_fwd": stage_ms[0] / pi, "stencil_gram_loss_adjoint": stage_ms[1] / pi,
          "mlp_bwd_reduce": stage_ms[2] / pi, "adam": stage_ms[3] / pi}
    # the dominant kernel: the fused forward (A1), one launch per Adam iteration; its algorithmic flops
    # are the forward third of SURVEY.md §8's count
    hid, Lh = w.widths[1], len(w.widths) - 2
    fwd_flops = 2.0 * (2 * hid + (Lh - 1) * hid * hid + hid) * w.points * tile_frac
    clocks = sampler.summary()
    line = {
        "metric": f"CRVPINN Adam iters/s ({args.workload})", "value": value, "unit": "Adam iters/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
        "higher_is_better": True, "scaling": "strong" if args.shard else "weak", "vs_baseline": None,
        "dtype": "f16" if prec == crv.PREC_TENSOR else "f32", "data": "synthetic",
        "config": dict(workload_config(args.workload, args.precision),
                       parallelism=f"points{world}" if args.shard else f"replicas{world}"),
        "points_iters_per_s": value * w.points,
        "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak,
                     "traffic": traffic.get(args.workload) if not args.shard else None,
                     "scope": "whole Adam iteration (A1-A8): SURVEY.md §8 algorithmic MLP flops per iteration / "
                              "device time per iteration of the timed region",
                     "alg_flops_per_iter": flops, "ms_per_iter": ms_iter, "peak_source": peak_note,
                     "traffic_source": traffic_src},
        "roofline_dominant_kernel": {
            "kernel": "k_tc_forward (A1, fused forward)" if prec == crv.PREC_TENSOR else "MLP forward (SIMT)",
            "achieved": fwd_flops / (st["mlp_fwd"] * 1e-3) / 1e12, "peak": peak, "unit": "TFLOP/s",
            "frac": fwd_flops / (st["mlp_fwd"] * 1e-3) / 1e12 / peak, "alg_flops_per_launch": fwd_flops,
            "us_per_launch": st["mlp_fwd"] * 1e3, "share_of_step": st["mlp_fwd"] / max(sum(st.values()), 1e-12),
            "timing": "CUDA event nodes on the library stream in a profiled replay of the same graph"},
        "stage_ms_per_iter": st,
        "clocks": clocks,
        "e2e": e2e,
        "gpu_launches": launches,
    }
    g.close()
    del S_dev
    if world == 1 and not args.shard and not args.no_per_workload:
        # C1..C5 (north_star: report every workload): device-timed it/s, points.it/s, ms/iter, roofline
        # fraction; the other four configs are timed with the same protocol, fewer steps
        per = {}
        for name in W.WORKLOADS:
            if name == args.workload:
                per[name] = {"it_s": value, "ms_per_iter": ms_iter}
            else:
                Fn = W.make_fields(name)
                wn = Fn.workload
                gn = crv.Crvpinn(wn.N, wn.widths, Fn.K, Fn.S, Fn.f, Fn.theta0, precision=prec, lr=wn.lr,
                                 device=local, stream=stream.cuda_stream)
                Sn = [torch.from_numpy(s).to(f"cuda:{local}") for s in Fn.S_steps]
                steps_n = max(3, min(args.steps, 10))
                tn, _ = time_steps(torch, gn, Sn, stream, flush, steps_n, max(3, min(args.warmup, 5)))
                gn.close()
                per[name] = {"it_s": steps_n * ITERS_PER_STEP / (tn / 1e3), "ms_per_iter": tn / (steps_n * ITERS_PER_STEP)}
            wn = W.WORKLOADS[name]
            per[name]["points_it_s"] = per[name]["it_s"] * wn.points
            ach, frac = roofline_frac(wn, per[name]["ms_per_iter"], peak)
            per[name]["roofline"] = {"achieved_tflops": ach, "frac": frac, "bound": bound,
                                     "traffic": traffic.get(name)}
        if not args.no_cpu_baseline:
            orc = time_oracle_table(list(W.WORKLOADS))
            for name, row in orc.items():
                per[name]["oracle"] = row
        line["per_workload"] = per
    if world == 1 and not args.no_cpu_baseline:
        n_or = 2
        v, cores, t_factor = time_oracle(args.workload, n_or)
        line["cpu_baseline"] = {"value": v, "unit": "Adam iters/s", "cores": cores, "kind": "oracle",
                                "cpu": cpu_model(),
                                "sample": f"{n_or} full Adam iterations of {args.workload} (fp64 oracle, OpenMP, "
                                          f"{cores} threads, right after the one-time LU factorisation "
                                          f"({t_factor:.1f}s, excluded))"}
    print(json.dumps(line), flush=True)
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
