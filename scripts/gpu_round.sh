#!/bin/bash
# Full measurement cycle for profiles/: tests, smoke, bench (C5 default + C4), ncu launch list of the
# bench command, ncu --set full of the top kernels. usage: scripts/gpu_round.sh <tag>
TAG=${1:-run}
mkdir -p gpurun_out
timeout -s KILL 400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_pytest_gpu.log 2>&1
timeout -s KILL 200 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout -s KILL 400 python bench.py > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err
timeout -s KILL 300 python bench.py --workload C4 --no-cpu-baseline > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
timeout -s KILL 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_plain.json 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
    > gpurun_out/${TAG}_ncu_launches.log 2>&1
timeout -s KILL 120 python scripts/prof_once.py C5 2 > gpurun_out/${TAG}_prof_plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_tc_forward|k_tc_bwd2|k_reduce|k_res_dst|k_tridiag|k_idst_loss|k_adj_final|k_tc_adam" -s 0 -c 16 \
    -o gpurun_out/${TAG}_full python scripts/prof_once.py C5 1 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo round-done
