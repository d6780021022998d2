# A/B timing: default library vs build/ab/<variant> (scripts/ab_build.sh); usage: xp_ab.sh <variant> [workload] [reps]
V=$1; W=${2:-C5}; R=${3:-3}
mkdir -p gpurun_out
for rep in $(seq $R); do for lib in default $V; do
  if [ $lib = default ]; then unset CRVPINN_LIB; else export CRVPINN_LIB=$PWD/build/ab/$lib/libcrvpinn.so; fi
  timeout -s KILL 200 python bench.py --workload $W --no-cpu-baseline --no-per-workload --no-e2e --steps 20 > /tmp/o.json 2>/dev/null
  python -c "import json;d=json.loads(open('/tmp/o.json').read().strip().splitlines()[-1]);print('$W $lib', round(d['value'],1), d['clocks']['sm_mhz'], d.get('stage_ms_per_iter'))" >> gpurun_out/xp_ab.log
done; done
unset CRVPINN_LIB
