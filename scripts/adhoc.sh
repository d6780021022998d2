#!/bin/bash
# A/B: default build vs variants under build/ab/ (stage times from the profiled step graph)
for r in 1 2; do
  for v in default clampn clampn_m6 clampn_m10 esleep; do
    if [ $v = default ]; then L=paper_2604_20731_b200/libcrvpinn.so; else L=build/ab/$v/libcrvpinn.so; fi
    CRVPINN_LIB=$L timeout 120 python scripts/stage_time.py C5 5 2>&1 | tail -1 | sed "s|^|$v: |"
  done
done
