#!/bin/bash
for v in nq4 nq1 h2s0 dsx1 mmas0; do
  CRVPINN_LIB=build/ab/$v/libcrvpinn.so timeout -s KILL 300 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "workload_theta0 and C5" 2>&1 | tail -1 | sed "s|^|$v |"
done
for r in 1 2 3; do
for v in base nq4 nq1 h2s0 dsx1 mmas0; do
  CRVPINN_LIB=build/ab/$v/libcrvpinn.so timeout -s KILL 120 python scripts/stage_time.py C5 3 2>&1 | tail -1 | sed "s|^|$v |"
done; done
