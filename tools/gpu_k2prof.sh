#!/bin/bash
# one ncu --set full capture of the K2 row-cost kernel on 1,000 C5 parents x 240 tilings
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cost_rows -s 1 -c 1 \
   -o gpurun_out/prof_k2 -f python tools/prof_k1.py 1000 > gpurun_out/ncu_full_k2.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_full_k2.log
exit 0
