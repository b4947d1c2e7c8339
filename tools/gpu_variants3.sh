#!/bin/bash
# Bench engine builds over sweep sizes (seeds 4, 8, 16).  Usage: bash tools/gpu_variants3.sh TAG a.so ...
TAG=$1; shift
OUT=gpurun_out
mkdir -p $OUT
LIB=paper_2506_18796_b200/lib/libcace_gpu.so
cp $LIB /tmp/orig.so
for v in "$@"; do
  name=$(basename $v .so)
  cp $v $LIB
  for sd in 4 8 16; do
    timeout 600 python bench.py --seeds $sd --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_${TAG}_${name}_s$sd.log 2>&1
  done
done
cp /tmp/orig.so $LIB
