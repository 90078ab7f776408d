#!/bin/bash
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
: > gpurun_out/variants_c2.txt
for nm in $names; do
  echo "== $nm" >> gpurun_out/variants_c2.txt
  GS_LIB_PATH=/tmp/lib_$nm.so timeout 600 python tools/bench_extras.py --only c2_unsharp c2_harris --no-cpu 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['workload'], round(d['candidates_per_s']), d['step_breakdown_ms']['featurize'])" >> gpurun_out/variants_c2.txt
done
