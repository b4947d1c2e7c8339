#!/bin/bash
# Full-occupancy ncu capture (source counters + stall reasons) of one replay kernel
# of the default config-4 bench.  Usage: bash tools/gpu_stall.sh TAG [CAPACITY]
TAG=${1:-stall}
CAP=${2:-5}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"replay_lane_kernel<.int.$CAP," -c 1 -o $OUT/prof_$TAG \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_$TAG.log 2>&1
echo "rc=$?" >> $OUT/ncu_$TAG.log
