#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/k1_stats.py 1000 > gpurun_out/k1_stats.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5.py tests/test_gpu_reuse.py -x -q -p no:cacheprovider > gpurun_out/pytest_k1ab.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_k1ab.log
