#!/bin/bash
# Copy one tools/gpu_final.sh run's artefacts from gpurun_out/ into tracked profiles/<tag>_* files.
tag=$1
set -e
python tools/summarize_profiles.py $tag k1 k2
grep '^{' gpurun_out/bench.log | tail -n 1 > profiles/${tag}_bench.json || true
grep '^{' gpurun_out/bench_ref.log | tail -n 1 > profiles/${tag}_bench_reference.json || true
cp gpurun_out/pytest_gpu.log profiles/${tag}_pytest_gpu.log
[ -s gpurun_out/search_b8.json ] && cp gpurun_out/search_b8.json profiles/${tag}_search_c3_b8p2.json
for t in memcheck racecheck synccheck; do
  [ -f gpurun_out/san2_$t.log ] && ! grep -q "is closed" gpurun_out/san2_$t.log && cp gpurun_out/san2_$t.log profiles/${tag}_san_$t.log
done
ls -la profiles/${tag}_*
