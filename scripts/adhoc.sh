#!/bin/bash
timeout -s KILL 700 python -m pytest tests -q -m gpu 2>&1 | tail -2
for w in C3 C4 C5; do for v in "CRVPINN_BWD_CHAIN=0" "X=1"; do
  env $v timeout -s KILL 120 python scripts/stage_time.py $w 5 2>&1 | tail -1 | sed "s|^|$w $v |"
done; done
