#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:featurize_kernel -s 1 -c 1 \
   -o gpurun_out/prof_k1 -f python tools/prof_k1.py 1000 > gpurun_out/ncu_full.log 2>&1
ncu -i gpurun_out/prof_k1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/k1_source.csv 2>/dev/null
ncu -i gpurun_out/prof_k1.ncu-rep --page raw --csv > gpurun_out/k1_raw.csv 2>/dev/null
exit 0
