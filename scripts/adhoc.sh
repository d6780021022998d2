timeout -s KILL 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r01v20_pytest.log 2>&1
timeout -s KILL 300 bash scripts/gpu_times.sh r01v20
