timeout -s KILL 300 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r01v31_pytest.log 2>&1
timeout -s KILL 200 python bench.py --no-cpu-baseline > gpurun_out/r01v31_bench.json 2> gpurun_out/r01v31_bench.err
