timeout -s KILL 120 python scripts/fwd_time.py C5 50 > gpurun_out/fwd_time25.log 2>&1
CRVPINN_LIB=$PWD/paper_2604_20731_b200/libexp_nolo.so timeout -s KILL 120 python scripts/fwd_time.py C5 50 >> gpurun_out/fwd_time25.log 2>&1
CRVPINN_LIB=$PWD/paper_2604_20731_b200/libexp_nolo.so CRVPINN_FWD_TRACE=gpurun_out/fwd_trace_nolo.bin timeout -s KILL 120 python scripts/fwd_time.py C5 3 > gpurun_out/trace.log 2>&1
