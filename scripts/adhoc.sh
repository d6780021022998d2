timeout 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r01v7_pytest.log 2>&1
timeout 200 python scripts/tc_check.py 0 > gpurun_out/r01v7_tc_check.log 2>&1
bash scripts/gpu_times.sh r01v7
