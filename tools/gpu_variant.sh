#!/bin/bash
# A/B of K1 build variants: VARIANTS="name:flags ..." (default build first)
mkdir -p gpurun_out
cp paper_2012_07145_b200/libgs_sched.so /tmp/lib_default.so
names="default"
for v in $VARIANTS; do
  name=${v%%:*}; flags=${v#*:}; flags=${flags//,/ }
  GS_NVCC_EXTRA="$flags" python -c "from paper_2012_07145_b200 import _build; _build.build(force=True)" > /dev/null 2> gpurun_out/build_$name.err
  cp paper_2012_07145_b200/libgs_sched.so /tmp/lib_$name.so
  names="$names $name"
done
cp /tmp/lib_default.so paper_2012_07145_b200/libgs_sched.so
: > gpurun_out/variants.txt
for rep in 1 2; do for nm in $names; do
  echo "== $nm" >> gpurun_out/variants.txt
  GS_LIB_PATH=/tmp/lib_$nm.so timeout 300 python tools/k1_stats.py ${PARENTS:-1000} 2>&1 | head -1 >> gpurun_out/variants.txt
done; done
