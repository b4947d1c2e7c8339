#!/bin/bash
# ncu source-level stall capture of one capacity kernel at LOW occupancy (4
# seeds: ~1 warp per scheduler), where stall samples expose the per-request
# dependency chain.  Usage: bash tools/gpu_stall_small.sh TAG CAPACITY
TAG=${1:-small}
CAP=${2:-6}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"replay_lane_kernel<.int.$CAP," -c 1 -o $OUT/prof_$TAG \
  python bench.py --seeds 4 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_$TAG.log 2>&1
echo "rc=$?" >> $OUT/ncu_$TAG.log
