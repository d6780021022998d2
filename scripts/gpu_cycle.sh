#!/bin/bash
# One GPU measurement cycle (run under gpurun): tests, smoke, bench C5/C4, ncu launch list.
# usage: scripts/gpu_cycle.sh <tag> [full]
TAG=${1:-run}
mkdir -p gpurun_out
timeout 240 python scripts/tc_check.py 0 > gpurun_out/${TAG}_tc_check.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 400 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench_c5.log 2>&1
timeout 200 python bench.py --workload C4 --no-cpu-baseline > gpurun_out/${TAG}_bench_c4.log 2>&1
if [ "$2" == "full" ]; then
  timeout 200 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/${TAG}_launches_c5.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
      > gpurun_out/${TAG}_ncu.log 2>&1
fi
echo cycle-done
