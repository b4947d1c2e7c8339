#!/bin/bash
# A/B of engine environment settings over sweep sizes, in-tree library.
# Usage: bash tools/gpu_ab_env.sh TAG "ENV1" "ENV2" ...   ("" = defaults)
# AB_ARGS overrides the workload list (';'-separated bench.py argument sets).
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
IFS=';' read -ra WL <<< "${AB_ARGS:---seeds 32;--seeds 16;--seeds 8;--seeds 4;--config 3}"
for envs in "$@"; do
  for args in "${WL[@]}"; do
    a=$(echo $args | tr -d ' -')
    env $envs timeout 900 python bench.py $args --steps 3 --warmup 3 --no-e2e --cpu-sample 0 --parity-sample 64 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('[$envs]', '$a', round(d['value']/1e9,2), round(d['ms_per_step'],1), 'launches', d['gpu_launches'], 'parity', (d.get('parity_sample') or {}).get('bit_exact'))" >> $OUT/ab_$TAG.txt
  done
done
