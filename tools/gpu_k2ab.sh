#!/bin/bash
# K2 A/B: DMMA row-cost kernel variants (build_ab/lib_*.so) against the default build and the scalar path
mkdir -p gpurun_out
: > gpurun_out/k2ab.txt
timeout 600 python -m pytest tests -x -q -m gpu -k "parity or c5 or reuse or cost or ops" > gpurun_out/k2_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/k2_tests.log
for rep in 1 2; do
  for v in default ${VARIANTS:-} scalar; do
    case $v in
      default) env="GS_X=1" ;;
      scalar) env="GS_K2_SCALAR=1" ;;
      *) env="GS_LIB_PATH=build_ab/lib_$v.so" ;;
    esac
    echo "== $v" >> gpurun_out/k2ab.txt
    env $env timeout 300 python bench.py --steps 3 --no-cpu --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['step_breakdown_ms'], d['parity']['ok'], d['parity']['rep_cost_max_rel_err'], d['parity']['sample_total_max_rel_err'])" >> gpurun_out/k2ab.txt 2>&1
  done
done
exit 0
