#!/bin/bash
# K1 compile-flag variants: build each into its own .so, time K1 on 240K C5 candidates
mkdir -p gpurun_out
: > gpurun_out/flags.txt
for v in "base:" "ptxO2:-Xptxas -O2" "ptxO1:-Xptxas -O1" "cicc2:-Xcicc -O2" "cicc1:-Xcicc -O1"; do
  name=${v%%:*}; flags=${v#*:}
  GS_NVCC_EXTRA="$flags" python -c "from paper_2012_07145_b200 import _build; _build.build(force=True)" > /dev/null 2>gpurun_out/build_$name.err || { echo "$name build failed" >> gpurun_out/flags.txt; continue; }
  cp paper_2012_07145_b200/libgs_sched.so /tmp/lib_$name.so
  echo "== $name ($flags)" >> gpurun_out/flags.txt
  GS_LIB_PATH=/tmp/lib_$name.so timeout 300 python tools/k1_stats.py 1000 2>&1 | head -2 >> gpurun_out/flags.txt
done
