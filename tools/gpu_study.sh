#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/row_memo_study.py 100 > gpurun_out/memo_study.txt 2>&1
timeout 600 python tools/k1_stats.py 1000 > gpurun_out/k1_stats.txt 2>&1
GS_NVCC_EXTRA=-DGS_PHASES timeout 600 python -c "from paper_2012_07145_b200 import _build; _build.build(force=True)" > gpurun_out/phases_build.txt 2>&1
timeout 600 python tools/k1_stats.py 1000 > gpurun_out/k1_phases.txt 2>&1
