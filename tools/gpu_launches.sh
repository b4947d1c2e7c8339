#!/bin/bash
# ncu launch list (per-launch duration + DRAM bytes, serialised) of one bench.py step.
# Usage: bash tools/gpu_launches.sh TAG [bench.py args...]
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
  --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline "$@" > $OUT/ncu_launch_$TAG.log 2>&1
echo "rc=$?" >> $OUT/ncu_launch_$TAG.log
