#!/bin/bash
CRVPINN_LIB=build/ab/swap/libcrvpinn.so timeout -s KILL 60 python scripts/outl_case.py 64 256 5 2>&1 | head -1
for r in 1 2 3; do
for v in default swap; do
  if [ $v = default ]; then L=paper_2604_20731_b200/libcrvpinn.so; else L=build/ab/$v/libcrvpinn.so; fi
  CRVPINN_LIB=$L timeout -s KILL 120 python scripts/stage_time.py C5 3 2>&1 | tail -1 | sed "s|^|$v |"
done; done
