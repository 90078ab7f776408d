#!/bin/bash
mkdir -p gpurun_out
cp paper_2012_07145_b200/libgs_sched.so /tmp/lib_default.so
GS_NVCC_EXTRA="-DGS_HEADS_FREE" python -c "from paper_2012_07145_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
cp paper_2012_07145_b200/libgs_sched.so /tmp/lib_hfree.so
cp /tmp/lib_default.so paper_2012_07145_b200/libgs_sched.so
: > gpurun_out/heads.txt
for rep in 1 2; do
for cfg in "default 0" "default 1" "hfree 0" "hfree 1"; do set -- $cfg
  echo "== $1 headsmall=$2" >> gpurun_out/heads.txt
  if [ $2 = 1 ]; then export GS_K1_HEAD_SMALL=1; else unset GS_K1_HEAD_SMALL; fi
  GS_LIB_PATH=/tmp/lib_$1.so timeout 300 python tools/k1_stats.py 4167 2>&1 | head -1 >> gpurun_out/heads.txt
done; done
