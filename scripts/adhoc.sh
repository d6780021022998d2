#!/bin/bash
for v in dxf dxf_nt1 nt1; do CRVPINN_LIB=build/ab/$v/libcrvpinn.so timeout -s KILL 60 python scripts/outl_case.py 64 256 5 2>&1 | head -1 | sed "s|^|$v |"; done
for r in 1 2; do
for v in default dxf dxf_nt1 nt1; do
  if [ $v = default ]; then L=paper_2604_20731_b200/libcrvpinn.so; else L=build/ab/$v/libcrvpinn.so; fi
  CRVPINN_LIB=$L timeout -s KILL 120 python scripts/stage_time.py C5 3 2>&1 | tail -1 | sed "s|^|$v |"
done; done
for v in dxf_nt1; do
CRVPINN_LIB=build/ab/$v/libcrvpinn.so CRVPINN_BWD_TRACE=gpurun_out/b2x.bin CRVPINN_BWD_TRACE_G=2 timeout -s KILL 120 python scripts/prof_once.py C5 2 > /dev/null 2>&1
echo "$v g=2 $(python scripts/bwd2_report.py gpurun_out/b2x.bin)"
done
