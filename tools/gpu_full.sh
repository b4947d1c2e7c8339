#!/bin/bash
# Full-size bench (BASELINE config 4) + full-occupancy ncu capture of one replay kernel.
TAG=${1:-full}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > $OUT/clocks_$TAG.csv &
SMI=$!
timeout 1200 python bench.py > $OUT/bench_full_$TAG.log 2>&1
echo "rc=$?" >> $OUT/bench_full_$TAG.log
kill $SMI
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"replay_lane_kernel<5," -c 1 -o $OUT/prof_full_$TAG \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1
echo "rc=$?" >> $OUT/ncu_full_$TAG.log
