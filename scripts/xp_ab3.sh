# A/B timing of several variants: xp_ab3.sh <workload> <reps> <variant>... ("default" = the package library)
W=$1; R=$2; shift 2
mkdir -p gpurun_out
for rep in $(seq $R); do for lib in "$@"; do
  if [ $lib = default ]; then unset CRVPINN_LIB; else export CRVPINN_LIB=$PWD/build/ab/$lib/libcrvpinn.so; fi
  timeout -s KILL 200 python bench.py --workload $W --no-cpu-baseline --no-per-workload --no-e2e --steps 20 > /tmp/o.json 2>/dev/null
  python -c "import json;d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]);print('$W $lib', round(d['value'],1), d['clocks']['sm_mhz'], {k: round(v*1e3,1) for k,v in d.get('stage_ms_per_iter').items()})" >> gpurun_out/xp_ab.log
done; done
unset CRVPINN_LIB
