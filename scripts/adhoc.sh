timeout -s KILL 60 python scripts/outl_case.py 128 256 3 > gpurun_out/outl_dbg4.log 2>&1
timeout -s KILL 60 python scripts/outl_case.py 256 256 4 >> gpurun_out/outl_dbg4.log 2>&1
timeout -s KILL 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r01v28_pytest.log 2>&1 && \
timeout -s KILL 200 bash scripts/gpu_times.sh r01v28
