#!/bin/bash
# tests + variant comparison + full-occupancy profile of the C=5 lane kernel.
OUT=gpurun_out
TAG=${TAG:-x}
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 -x > $OUT/pytest_gpu_$TAG.log 2>&1
echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
bash tools/gpu_exp.sh "$@"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:replay_lane_kernel<\(int\)5' -c 1 -o $OUT/prof_full_$TAG \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1
echo "rc=$?" >> $OUT/ncu_full_$TAG.log
