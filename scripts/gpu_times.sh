#!/bin/bash
# Bench line + per-kernel durations (ncu launch list of one eager loss_grad). usage: scripts/gpu_times.sh <tag> [workload]
TAG=${1:-run}
WL=${2:-C5}
mkdir -p gpurun_out
timeout 300 python bench.py --no-cpu-baseline --no-e2e --workload ${WL} ${BENCH_ARGS} > gpurun_out/${TAG}_bench.log 2>&1
timeout 300 python scripts/prof_once.py ${WL} 2 > gpurun_out/${TAG}_prof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv python scripts/prof_once.py ${WL} 2 > gpurun_out/${TAG}_ncu.log 2>&1
echo times-done
