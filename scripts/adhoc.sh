#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "iga" > gpurun_out/pt.log 2>&1; tail -3 gpurun_out/pt.log
timeout -s KILL 600 python scripts/iga_accuracy.py
CRVPINN_IGA_BAND=reg timeout -s KILL 600 python scripts/iga_accuracy.py
timeout -s KILL 600 python scripts/bench_iga.py > gpurun_out/iga.json 2>gpurun_out/iga.err; tail -c 900 gpurun_out/iga.json; tail -3 gpurun_out/iga.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/iga_launches.csv python scripts/prof_iga.py > gpurun_out/ncu.log 2>&1
