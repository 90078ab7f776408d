#!/bin/bash
# iteration: GPU tests (stop at first failure), K1 stats, short bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/k1_stats.py 1000 > gpurun_out/k1_stats.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-extras > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench rc=$?" >> gpurun_out/bench.err
