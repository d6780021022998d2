"""bench.py host logic on CPU: the reference arm's JSON line (the oracle timed as the reference,
tier contract), the algorithmic work the roofline divides by, and that our arm
fails loudly without a GPU instead of falling back to the CPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"]


def _run(*args, timeout=600):
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=timeout, cwd=ROOT)


def test_reference_arm_json_line():
    r = _run("--impl", "reference", "--workload", "C1", "--steps", "3", "--warmup", "1")
    assert r.returncode == 0, r.stderr
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in REQUIRED:
        assert k in d, k
    assert d["impl"] == "reference" and d["dtype"] == "f64" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 3 and d["warmup"] == 1
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["workload"].startswith("C1") and "1 per step" in d["cpu_baseline"]["sample"]


def test_algorithmic_work_matches_design():
    import bench
    import workloads as W
    # 4.116e11 flops per Adam iteration at C5, 2.57e10 at C4
    assert abs(bench.alg_flops_per_iter(W.WORKLOADS["C5"]) - 4.116e11) / 4.116e11 < 1e-3
    assert abs(bench.alg_flops_per_iter(W.WORKLOADS["C4"]) - 2.57e10) / 2.57e10 < 2e-3
    assert 1.5e7 < bench.alg_bytes_per_iter(W.WORKLOADS["C5"]) < 3e7


def test_our_arm_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = _run("--workload", "C1", "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--no-e2e", timeout=300)
    assert r.returncode != 0
    assert not any(ln.startswith("{") for ln in r.stdout.splitlines())
