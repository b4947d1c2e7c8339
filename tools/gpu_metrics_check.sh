#!/bin/bash
# RunMetrics pipeline: GPU tests, phase timing (32 and 4 seeds), launch list of a 4-seed call.
TAG=${1:-mc}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 -x > $OUT/pytest_gpu_$TAG.log 2>&1
echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
CACE_TIMING=1 timeout 600 python tools/metrics_timing.py 32 > $OUT/metrics_$TAG.log 2>&1
CACE_TIMING=1 timeout 600 python tools/metrics_timing.py 4 >> $OUT/metrics_$TAG.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_metrics_$TAG.csv \
  python tools/metrics_timing.py 4 > $OUT/ncu_metrics_$TAG.log 2>&1
echo "rc=$?" >> $OUT/ncu_metrics_$TAG.log
