#!/bin/bash
# Quick GPU check: tc_check numerics, pytest -m gpu, C5 bench line. usage: scripts/gpu_quick.sh <tag>
TAG=${1:-run}
mkdir -p gpurun_out
timeout 240 python scripts/tc_check.py 0 > gpurun_out/${TAG}_tc_check.log 2>&1
echo "tc_check rc=$?" >> gpurun_out/${TAG}_tc_check.log
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_pytest.log 2>&1
timeout 300 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/${TAG}_bench_c5.log 2>&1
echo quick-done
