timeout -s KILL 60 python scripts/outl_case.py 256 256 4 > gpurun_out/e16.log 2>&1
timeout -s KILL 200 bash scripts/gpu_times.sh r01v37
CRVPINN_LIB=$PWD/paper_2604_20731_b200/libexp_e8.so timeout -s KILL 200 bash scripts/gpu_times.sh r01v37e8
