#!/bin/bash
timeout -s KILL 60 python scripts/outl_case.py 64 256 5 2>&1 | head -1
CRVPINN_BWD_CHAIN=0 timeout -s KILL 60 python scripts/outl_case.py 64 256 5 2>&1 | head -1
for r in 1 2; do
for v in "CRVPINN_BWD_CHAIN=0" "CRVPINN_BWD_STAGES=4" "CRVPINN_BWD_STAGES=2" "CRVPINN_BWD_STAGES=1"; do
  env $v timeout -s KILL 120 python scripts/stage_time.py C5 3 2>&1 | tail -1 | sed "s|^|$v |"
done
CRVPINN_LIB=build/ab/tlast/libcrvpinn.so CRVPINN_BWD_CHAIN=0 timeout -s KILL 120 python scripts/stage_time.py C5 3 2>&1 | tail -1 | sed "s|^|tlast bwd2 |"
done
timeout -s KILL 120 python scripts/chain_trace.py C5 > /dev/null 2>&1
