#!/bin/bash
# per-launch K1 times of prebuilt libraries: LIBS="a.so b.so" (ncu launch durations, relative use only)
mkdir -p gpurun_out
: > gpurun_out/launch_ab.txt
for l in $LIBS; do
  echo "== $l" >> gpurun_out/launch_ab.txt
  GS_LIB_PATH=$l timeout 300 python tools/k1_stats.py ${PARENTS:-4167} 2>&1 | head -1 >> gpurun_out/launch_ab.txt
  GS_LIB_PATH=$l timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:featurize_kernel --csv python tools/k1_stats.py ${PARENTS:-4167} 2>/dev/null | grep featurize_kernel | awk -F'","' '{print $NF}' | tr -d '"' | head -4 | tr '\n' ' ' >> gpurun_out/launch_ab.txt
  echo >> gpurun_out/launch_ab.txt
done
