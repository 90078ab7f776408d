#!/bin/bash
mkdir -p gpurun_out
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/sanitize_step.py > gpurun_out/san_blocking.log 2>&1; echo "rc=$?" >> gpurun_out/san_blocking.log
for tool in racecheck synccheck; do
 for sz in 720 9600; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_step.py $sz > gpurun_out/san_${tool}_$sz.log 2>&1
  echo "rc=$?" >> gpurun_out/san_${tool}_$sz.log
 done
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_step.py > gpurun_out/san_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/san_memcheck.log
timeout 900 python -m pytest tests/test_gpu_ops.py -x -q -p no:cacheprovider > gpurun_out/pytest_ops.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ops.log
