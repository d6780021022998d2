#!/bin/bash
for r in 1 2; do
for v in default tfirst; do
  if [ $v = default ]; then L=paper_2604_20731_b200/libcrvpinn.so; else L=build/ab/$v/libcrvpinn.so; fi
  CRVPINN_LIB=$L timeout -s KILL 120 python scripts/stage_time.py C5 3 2>&1 | tail -1 | sed "s|^|$v |"
done; done
CRVPINN_LIB=build/ab/tfirst/libcrvpinn.so CRVPINN_BWD_TRACE=gpurun_out/b2f.bin CRVPINN_BWD_TRACE_G=2 timeout -s KILL 120 python scripts/prof_once.py C5 2 > /dev/null 2>&1
echo "tfirst g=2 $(python scripts/bwd2_report.py gpurun_out/b2f.bin)"
