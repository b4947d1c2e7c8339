#!/bin/bash
# ncu --set full capture (source counters + stalls) of the first launch matching
# a kernel regex in one bench.py step; writes gpurun_out/prof_TAG.ncu-rep.
# Usage: bash tools/gpu_ncu.sh TAG REGEX [bench.py args...]
TAG=$1; RE=$2; shift 2
OUT=gpurun_out; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"$RE" -c 1 -o $OUT/prof_$TAG -f \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline "$@" > $OUT/ncu_$TAG.log 2>&1
echo "rc=$?" >> $OUT/ncu_$TAG.log
