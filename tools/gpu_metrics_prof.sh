#!/bin/bash
# RunMetrics path: phase timings (32 and 4 seeds) + launch list of one 4-seed call.
TAG=${1:-m}
OUT=gpurun_out
mkdir -p $OUT
CACE_TIMING=1 timeout 600 python tools/metrics_timing.py 32 > $OUT/metrics_$TAG.log 2>&1
CACE_TIMING=1 timeout 600 python tools/metrics_timing.py 4 >> $OUT/metrics_$TAG.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum --clock-control none --csv --log-file $OUT/launches_metrics_$TAG.csv \
  python tools/metrics_timing.py 4 > $OUT/ncu_metrics_$TAG.log 2>&1
echo "rc=$?" >> $OUT/ncu_metrics_$TAG.log
