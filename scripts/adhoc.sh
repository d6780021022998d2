timeout -s KILL 120 python scripts/tc_check.py 0 > gpurun_out/r01v18_tc.log 2>&1; echo "rc=$?" >> gpurun_out/r01v18_tc.log
CRVPINN_FWD_TRACE=gpurun_out/fwd_trace18.bin timeout -s KILL 120 python scripts/prof_once.py C5 1 > gpurun_out/trace.log 2>&1
