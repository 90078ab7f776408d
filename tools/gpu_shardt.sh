#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_shard.py tests/test_gpu_search.py -x -q -p no:cacheprovider > gpurun_out/pytest_shard.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_shard.log
