#!/bin/bash
# A/B engine builds: config 4 at 1M and 131k scenarios (+ latency mode off), config 3.
# Usage: bash tools/gpu_variants.sh TAG a.so b.so ...   (the in-tree library is "base")
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
LIB=paper_2506_18796_b200/lib/libcace_gpu.so
cp $LIB /tmp/base.so
for v in /tmp/base.so "$@"; do
  name=$(basename $v .so)
  cp $v $LIB
  for args in "--seeds 32" "--seeds 4" "--config 3"; do
    a=$(echo $args | tr -d ' -')
    timeout 600 python bench.py $args --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$name', '$a', 'lat=on', round(d['value']/1e9,2), round(d['ms_per_step'],1))" >> $OUT/variants_$TAG.txt
    CACE_LATENCY_WAVES=0 timeout 600 python bench.py $args --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$name', '$a', 'lat=off', round(d['value']/1e9,2), round(d['ms_per_step'],1))" >> $OUT/variants_$TAG.txt
  done
done
cp /tmp/base.so $LIB
