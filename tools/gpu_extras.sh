#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python tools/bench_extras.py > gpurun_out/extras.jsonl 2> gpurun_out/extras.err
echo "rc=$?" >> gpurun_out/extras.err
