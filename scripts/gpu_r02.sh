#!/bin/bash
# Round-2 GPU cycle: usage scripts/gpu_r02.sh <tag> [what...]; what in {tests, smoke, bench, bench4, probe, launches, full}
TAG=${1:-run}; shift
WHAT=${@:-tests smoke bench}
mkdir -p gpurun_out
for w in $WHAT; do case $w in
tests) timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/${TAG}_pytest_gpu.log 2>&1 ;;
smoke) timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1 ;;
bench) timeout -s KILL 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err ;;
benchq) timeout -s KILL 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err ;;
bench4) timeout -s KILL 300 python bench.py --workload C4 --no-cpu-baseline --no-per-workload > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err ;;
probe) timeout -s KILL 300 python scripts/c3_grad_error.py > gpurun_out/${TAG}_probe.log 2>&1 ;;
launches) timeout -s KILL 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-per-workload > gpurun_out/${TAG}_plain.json 2>&1 && \
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-per-workload \
    > gpurun_out/${TAG}_ncu_launches.log 2>&1 ;;
full) timeout -s KILL 120 python scripts/prof_once.py C5 2 > gpurun_out/${TAG}_prof_plain.log 2>&1 && \
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_tc_|k_reduce|k_res_dst|k_tridiag|k_idst_loss|k_adj_final" -s 0 -c 16 \
    -o gpurun_out/${TAG}_full python scripts/prof_once.py C5 1 > gpurun_out/${TAG}_ncu_full.log 2>&1 ;;
esac; done
echo cycle-done
