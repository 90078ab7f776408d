#!/bin/bash
# A/B of prebuilt libraries: LIBS="build_ab/lib_old.so build_ab/lib_new.so", PARENTS (default 4167 = the 1M C5 step)
mkdir -p gpurun_out
: > gpurun_out/ab.txt
for rep in 1 2 3; do for l in ${LIBS:-build_ab/lib_old.so build_ab/lib_new.so}; do
  echo "== $l" >> gpurun_out/ab.txt
  GS_LIB_PATH=$l timeout 300 python tools/k1_stats.py ${PARENTS:-4167} 2>&1 | head -2 >> gpurun_out/ab.txt
done; done
