#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_phase1.py -x -q -p no:cacheprovider > gpurun_out/pytest_p1.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_p1.log
