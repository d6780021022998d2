#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "direct_solve" > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
timeout -s KILL 600 python scripts/bench_direct_solve.py > gpurun_out/ds.json 2>gpurun_out/ds.err; tail -c 1500 gpurun_out/ds.json; tail -3 gpurun_out/ds.err
