#!/bin/bash
# ncu --set full capture of the MLP kernels on C5 (one eager loss_grad after one warm-up).
# usage: scripts/ncu_full.sh <tag> [kernel-regex] [count]
TAG=${1:-run}
RE=${2:-"k_tc_forward|k_tc_bwd_layer|k_reduce|k_tc_out_bwd"}
CNT=${3:-7}
mkdir -p gpurun_out
timeout 300 python scripts/prof_once.py C5 2 > gpurun_out/${TAG}_prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${RE}" -s 0 -c ${CNT} \
    -o gpurun_out/${TAG}_full python scripts/prof_once.py C5 1 > gpurun_out/${TAG}_ncu_full.log 2>&1
echo ncu-done $?
