#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_search.py -x -q -p no:cacheprovider > gpurun_out/pytest_search.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_search.log
timeout 900 python tools/search_timing.py --beam 2 --passes 1 --no-cpu > gpurun_out/st1.json 2>gpurun_out/st1.err
timeout 1200 python tools/search_timing.py --beam 8 --passes 2 --no-cpu > gpurun_out/st2.json 2>>gpurun_out/st1.err
