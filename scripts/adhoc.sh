#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "intermediates or direct_solve or workload_theta0 or maximum" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
for r in 1 2; do timeout -s KILL 120 python scripts/stage_time.py C5 3 2>&1 | tail -1; done
timeout -s KILL 600 python scripts/bench_direct_solve.py --no-oracle > gpurun_out/ds.json 2>&1; tail -c 400 gpurun_out/ds.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ds_launches.csv python scripts/prof_direct_solve.py > gpurun_out/ncu.log 2>&1
