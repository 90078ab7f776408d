#!/bin/bash
# A/B of K1 launch-shape overrides: ENVS="NAME=v,NAME2=v2 ..." ("-" = defaults); PARENTS (default 4167)
mkdir -p gpurun_out
: > gpurun_out/env_ab.txt
for rep in 1 2; do for e in ${ENVS:--}; do
  echo "== $e" >> gpurun_out/env_ab.txt
  if [ "$e" = "-" ]; then envs=""; else envs=${e//,/ }; fi
  env $envs timeout 300 python tools/k1_stats.py ${PARENTS:-4167} 2>&1 | sed -n '1p;4p' >> gpurun_out/env_ab.txt
done; done
