#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "eval_points or iga_buoyancy or gravity" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
timeout -s KILL 600 python scripts/bench_eval_points.py > gpurun_out/ep.json 2>&1; tail -c 600 gpurun_out/ep.json
