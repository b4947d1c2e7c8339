#!/bin/bash
# Parity + bench + launch list + one full ncu capture of the C=5 replay kernel.
TAG=${1:-it}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 -x > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python bench.py --requests 20000 --seeds 4 --steps 3 --warmup 3 --e2e-steps 1 --cpu-sample 16 > $OUT/bench_small_$TAG.log 2>&1
echo "rc=$?" >> $OUT/bench_small_$TAG.log
timeout 600 python bench.py --requests 100000 --seeds 8 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_mid_$TAG.log 2>&1
echo "rc=$?" >> $OUT/bench_mid_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__inst_executed.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --requests 20000 --seeds 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
echo "rc=$?" >> $OUT/ncu_launch_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_lane_kernel -s 4 -c 1 -o $OUT/prof_$TAG \
  python bench.py --requests 20000 --seeds 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1
echo "rc=$?" >> $OUT/ncu_full_$TAG.log
