#!/bin/bash
# A/B: K1 default vs lockstep diagnostic variants (-DGS_LOCKSTEP=1,2,3)
mkdir -p gpurun_out
cp paper_2012_07145_b200/libgs_sched.so /tmp/lib_default.so
for v in 1 2 3; do
  GS_NVCC_EXTRA="-DGS_LOCKSTEP=$v" python -c "from paper_2012_07145_b200 import _build; _build.build(force=True)" > /dev/null 2> gpurun_out/build_ls$v.err
  cp paper_2012_07145_b200/libgs_sched.so /tmp/lib_ls$v.so
done
cp /tmp/lib_default.so paper_2012_07145_b200/libgs_sched.so
: > gpurun_out/lockstep.txt
for v in default ls1 ls2 ls3 default ls1 ls2 ls3; do
  echo "== $v" >> gpurun_out/lockstep.txt
  GS_LIB_PATH=/tmp/lib_$v.so timeout 300 python tools/k1_stats.py 1000 2>&1 | head -1 >> gpurun_out/lockstep.txt
done
