#!/bin/bash
timeout -s KILL 60 python scripts/outl_case.py 64 256 5 2>&1 | head -9
timeout -s KILL 700 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for r in 1 2 3; do
for v in default prev; do
  if [ $v = default ]; then L=paper_2604_20731_b200/libcrvpinn.so; else L=build/ab/$v/libcrvpinn.so; fi
  CRVPINN_LIB=$L timeout -s KILL 120 python scripts/stage_time.py C5 3 2>&1 | tail -1 | sed "s|^|$v |"
done; done
for g in 3 2 0; do
  CRVPINN_BWD_TRACE=gpurun_out/b2m_$g.bin CRVPINN_BWD_TRACE_G=$g timeout -s KILL 120 python scripts/prof_once.py C5 2 > /dev/null 2>&1
  echo "g=$g $(python scripts/bwd2_report.py gpurun_out/b2m_$g.bin)"
done
