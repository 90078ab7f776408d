#!/bin/bash
# Round-2 measurement: GPU parity tests, full bench line (CPU reference beside it), the reference
# arm, ncu launch list, ncu full captures of K1/K2, and the C3 search wall time (both arms).
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-extras > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:featurize_kernel -s 1 -c 1 \
   -o gpurun_out/prof_k1 -f python tools/prof_k1.py 1000 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cost_rows -s 1 -c 1 \
   -o gpurun_out/prof_k2 -f python tools/prof_k1.py 1000 > gpurun_out/ncu_full_k2.log 2>&1
timeout 1200 python tools/search_timing.py --beam 8 --passes 2 > gpurun_out/search_b8.json 2> gpurun_out/search_b8.err
exit 0
