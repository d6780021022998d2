#!/bin/bash
# A/B: side-stream weight reduction on/off, alternating
for r in 1 2 3; do
  for v in 1 0; do
    CRVPINN_SIDE_REDUCE=$v timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}_${r}.log 2>&1
    echo "side=$v run=$r $(python -c "import json,sys; d=json.loads(open('gpurun_out/ab_${v}_${r}.log').read().strip().splitlines()[-1]); print(round(d['value'],1), d['clocks']['sm_mhz'])")"
  done
done
