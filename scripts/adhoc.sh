#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -x -q -m gpu > gpurun_out/pt.log 2>&1; tail -15 gpurun_out/pt.log
for r in 1 2; do timeout -s KILL 120 python scripts/stage_time.py C5 3 2>&1 | tail -1; done
