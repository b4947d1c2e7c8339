#!/bin/bash
# Quick iteration: GPU parity tests, config-4 bench (device value only), launch list.
TAG=${1:-q}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 -x > $OUT/pytest_gpu_$TAG.log 2>&1
echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_$TAG.log 2>&1
echo "rc=$?" >> $OUT/bench_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.per_cycle_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
echo "rc=$?" >> $OUT/ncu_launch_$TAG.log
