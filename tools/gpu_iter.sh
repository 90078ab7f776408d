#!/bin/bash
# Iteration check: GPU parity tests, K1 counters/timing, short bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/k1_stats.py 1000 > gpurun_out/k1_stats.log 2>&1
timeout 900 python bench.py --steps 3 --no-cpu > gpurun_out/bench_quick.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_quick.log
exit 0
