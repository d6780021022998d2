#!/bin/bash
timeout -s KILL 600 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "workload_100 or nonfinite or checkpoint or zero_problem or composition" 2>&1 | tail -1
for r in 1 2 3; do
for v in base new; do
  if [ $v = new ]; then L=paper_2604_20731_b200/libcrvpinn.so; else L=build/ab/$v/libcrvpinn.so; fi
  CRVPINN_LIB=$L timeout -s KILL 120 python scripts/stage_time.py C5 3 2>&1 | tail -1 | sed "s|^|$v |"
done; done
