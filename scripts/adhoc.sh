#!/bin/bash
CRVPINN_LIB=build/ab/deep/libcrvpinn.so timeout -s KILL 300 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "C5 or C4 or chain or c3" 2>&1 | tail -3
for r in 1 2 3; do
for v in base deep; do
  L=build/ab/$v/libcrvpinn.so
  CRVPINN_LIB=$L timeout -s KILL 120 python scripts/stage_time.py C5 3 2>&1 | tail -2 | sed "s|^|$v |"
  CRVPINN_LIB=$L timeout -s KILL 120 python scripts/stage_time.py C4 3 2>&1 | tail -1 | sed "s|^|$v C4 |"
done; done
