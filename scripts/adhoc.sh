#!/bin/bash
mkdir -p gpurun_out
for wl in C5 C3; do
  timeout -s KILL 120 python scripts/coop_check.py $wl ${wl}_base 2>&1 | tail -1
  CRVPINN_FIELD_COOP=1 timeout -s KILL 120 python scripts/coop_check.py $wl ${wl}_coop 2>&1 | tail -3
done
python -c "
import numpy as np
for wl in ('C5','C3'):
    a=np.load('gpurun_out/'+wl+'_base.npy'); b=np.load('gpurun_out/'+wl+'_coop.npy')
    print(wl, 'bitwise', np.array_equal(a,b), 'maxdiff', float(np.abs(a-b).max()))
"
CRVPINN_FIELD_COOP=1 timeout -s KILL 600 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "intermediates or workload or gravity or composition" 2>&1 | tail -1
for r in 1 2 3; do
for v in base coop; do
  if [ $v = coop ]; then E="CRVPINN_FIELD_COOP=1"; else E="X=1"; fi
  env $E timeout -s KILL 120 python scripts/stage_time.py C5 3 2>&1 | tail -1 | sed "s|^|$v |"
done; done
