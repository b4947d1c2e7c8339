#!/bin/bash
# A/B of engine environment settings over sweep sizes.
# Usage: bash tools/gpu_ab_env.sh TAG "ENV1" "ENV2" ...   (e.g. "CACE_SPL=1" "CACE_SPL=2"; "" = defaults)
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
for envs in "$@"; do
  for args in "--seeds 32" "--seeds 16" "--seeds 8" "--seeds 4" "--config 3"; do
    a=$(echo $args | tr -d ' -')
    env $envs timeout 600 python bench.py $args --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('[$envs]', '$a', round(d['value']/1e9,2), round(d['ms_per_step'],1))" >> $OUT/ab_$TAG.txt
  done
done
