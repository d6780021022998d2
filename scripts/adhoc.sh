#!/bin/bash
for v in default msleep; do
  if [ $v = default ]; then L=paper_2604_20731_b200/libcrvpinn.so; else L=build/ab/$v/libcrvpinn.so; fi
  CRVPINN_LIB=$L timeout -s KILL 120 python scripts/stage_time.py C5 3 2>&1 | tail -1 | sed "s|^|$v |"
  for g in 3 2 0; do
    CRVPINN_LIB=$L CRVPINN_BWD_TRACE=gpurun_out/b2_$v_$g.bin CRVPINN_BWD_TRACE_G=$g timeout -s KILL 120 python scripts/prof_once.py C5 2 > /dev/null 2>&1
    echo "$v g=$g $(python scripts/bwd2_report.py gpurun_out/b2_$v_$g.bin)"
  done
done
