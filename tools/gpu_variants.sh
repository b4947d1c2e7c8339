#!/bin/bash
# Bench alternative builds of the engine library: bash tools/gpu_variants.sh TAG exp/a.so exp/b.so ...
# (each replaces lib/libcace_gpu.so for one config-4 bench + launch list; the original is restored)
TAG=$1; shift
OUT=gpurun_out
mkdir -p $OUT
LIB=paper_2506_18796_b200/lib/libcace_gpu.so
cp $LIB /tmp/orig.so
for v in base "$@"; do
  name=$(basename $v .so)
  if [ "$v" != base ]; then cp $v $LIB; else cp /tmp/orig.so $LIB; fi
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_${TAG}_$name.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.per_cycle_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file $OUT/launches_${TAG}_$name.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
cp /tmp/orig.so $LIB
