#!/bin/bash
# ncu --set full capture (source counters + stalls) of the first launch matching
# a kernel regex in one bench.py step.  Exports the raw metrics and the
# source/SASS page as CSV next to it (gpurun_out/ncu_TAG_{raw,src}.csv) and
# drops the .ncu-rep unless KEEP=1 (the reports exceed gpurun's 64 MiB).
# Usage: bash tools/gpu_ncu.sh TAG REGEX [bench.py args...]
TAG=$1; RE=$2; shift 2
OUT=gpurun_out; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"$RE" -c 1 -o $OUT/prof_$TAG -f \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline "$@" > $OUT/ncu_$TAG.log 2>&1
echo "rc=$?" >> $OUT/ncu_$TAG.log
if [ -f $OUT/prof_$TAG.ncu-rep ]; then
  ncu -i $OUT/prof_$TAG.ncu-rep --page raw --csv > $OUT/ncu_${TAG}_raw.csv 2>&1
  ncu -i $OUT/prof_$TAG.ncu-rep --page details --csv > $OUT/ncu_${TAG}_details.csv 2>&1
  ncu -i $OUT/prof_$TAG.ncu-rep --page source --csv --print-source cuda,sass > $OUT/ncu_${TAG}_src.csv 2>&1
  gzip -f $OUT/ncu_${TAG}_src.csv
  [ "$KEEP" = "1" ] || rm -f $OUT/prof_$TAG.ncu-rep
fi
