#!/bin/bash
# Compare kernel-library variants on the full config-4 bench (device value only).
OUT=gpurun_out
mkdir -p $OUT
for lib in "$@"; do
  name=$(basename $lib .so)
  CACE_GPU_LIB=$PWD/$lib timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > $OUT/exp_$name.log 2>&1
  echo "rc=$?" >> $OUT/exp_$name.log
done
