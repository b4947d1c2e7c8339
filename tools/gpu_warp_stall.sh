#!/bin/bash
# Full ncu capture of the warp-per-scenario kernel on a config-5 slice.
TAG=${1:-wstall}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"replay_warp_kernel" -c 1 -o $OUT/prof_$TAG \
  python bench.py --config 5 --requests 200000 --scenarios 2048 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_$TAG.log 2>&1
echo "rc=$?" >> $OUT/ncu_$TAG.log
