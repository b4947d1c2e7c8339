#!/bin/bash
# A/B of engine builds (CACE_GPU_LIB) over sweep sizes; one line per (lib, workload).
# Usage: bash tools/gpu_ab_libs.sh TAG LIB1 LIB2 ...   ("default" = the in-tree library)
# AB_ARGS overrides the workload list (';'-separated bench.py argument sets).
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
IFS=';' read -ra WL <<< "${AB_ARGS:---seeds 32;--seeds 4;--config 3}"
for lib in "$@"; do
  L=""; [ "$lib" != "default" ] && L="CACE_GPU_LIB=$PWD/$lib"
  for args in "${WL[@]}"; do
    a=$(echo $args | tr -d ' -')
    env $L timeout 900 python bench.py $args --steps 3 --warmup 3 --no-e2e --cpu-sample 0 --parity-sample 64 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$a', round(d['value']/1e9,2), round(d['ms_per_step'],1), 'parity', (d.get('parity_sample') or {}).get('bit_exact'))" >> $OUT/ab_$TAG.txt
  done
done
