#!/bin/bash
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_step.py > gpurun_out/san2_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/san2_$tool.log
done
