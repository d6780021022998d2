#!/bin/bash
mkdir -p gpurun_out
timeout -s KILL 600 /usr/local/cuda/bin/compute-sanitizer --print-limit 5 python -m pytest tests/test_parity_gpu.py -x -q -m gpu -k "test_intermediates_vs_oracle and 32-widths1-1-tensor" > gpurun_out/san.log 2>&1; grep -v "^    " gpurun_out/san.log | head -60
