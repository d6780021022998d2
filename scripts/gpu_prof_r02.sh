#!/bin/bash
# Round-2 profiling: ncu --set full of one eager loss_grad per workload (C5, C4, C3) -> per-kernel summary
# (scripts/ncu_summary.py), DRAM traffic per iteration (scripts/ncu_traffic.py) and the source-line page of
# the forward; the .ncu-rep files stay on the box (too large to bring back). Then the ncu launch list of
# the default bench command's timed step (C5). usage: scripts/gpu_prof_r02.sh <tag>
TAG=${1:-r02}
mkdir -p gpurun_out /tmp/ncu
K='regex:k_tc_forward|k_tc_bwd|k_tc_out|k_reduce|k_res_dst|k_tridiag|k_idst_loss|k_adj_final'
ARGS=""
for W in C5 C4 C3; do
  timeout -s KILL 120 python scripts/prof_once.py $W 1 > gpurun_out/${TAG}_prof_plain_$W.log 2>&1 && \
  timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k "$K" \
     -o /tmp/ncu/${TAG}_full_$W python scripts/prof_once.py $W 1 > gpurun_out/${TAG}_ncu_full_$W.log 2>&1
  python scripts/ncu_summary.py /tmp/ncu/${TAG}_full_$W.ncu-rep > gpurun_out/${TAG}_ncu_full_summary_$W.md 2>&1
  ARGS="$ARGS $W=/tmp/ncu/${TAG}_full_$W.ncu-rep"
done
python scripts/ncu_traffic.py $ARGS gpurun_out/${TAG}_traffic.json > gpurun_out/${TAG}_traffic.log 2>&1
ncu -i /tmp/ncu/${TAG}_full_C5.ncu-rep -k regex:k_tc_forward --page details --csv > gpurun_out/${TAG}_fwd_details_C5.csv 2>&1
timeout -s KILL 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-per-workload > gpurun_out/${TAG}_plain.json 2>&1 && \
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
    --no-per-workload > gpurun_out/${TAG}_ncu_launches.log 2>&1
du -sh gpurun_out
echo prof-done
