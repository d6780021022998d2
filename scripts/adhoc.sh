#!/bin/bash
timeout -s KILL 600 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "iga" 2>&1 | tail -1
timeout -s KILL 600 python scripts/bench_iga.py 2>&1 | tail -c 330
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/iga_launches.csv python scripts/prof_iga.py > gpurun_out/ncu.log 2>&1
