#!/bin/bash
# A/B of engine builds (CACE_GPU_LIB) over sweep sizes; one line per (lib, env, workload).
# Usage: bash tools/gpu_ab_libs.sh TAG LIB1 LIB2 ...   ("default" = the in-tree library)
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
for lib in "$@"; do
  L=""; [ "$lib" != "default" ] && L="CACE_GPU_LIB=$PWD/$lib"
  for envs in "" "CACE_LATENCY_WAVES=0"; do
    for args in "--seeds 32" "--seeds 4" "--config 3"; do
      [ "$envs" != "" ] && [ "$args" == "--seeds 32" ] && continue
      a=$(echo $args | tr -d ' -')
      env $L $envs timeout 600 python bench.py $args --steps 3 --warmup 3 --no-e2e --cpu-sample 0 --parity-sample 64 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '[$envs]', '$a', round(d['value']/1e9,2), round(d['ms_per_step'],1), 'parity', (d.get('parity_sample') or {}).get('bit_exact'))" >> $OUT/ab_$TAG.txt
    done
  done
done
