#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_c3.py -x -q -p no:cacheprovider > gpurun_out/pytest_c3.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_c3.log
timeout 1200 python tools/search_timing.py --beam 32 --passes 5 --no-cpu > gpurun_out/search_b32.json 2> gpurun_out/search_b32.err
