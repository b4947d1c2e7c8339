#!/bin/bash
# ncu --set full of one metrics_select_kernel launch (config 4, 4 seeds).
OUT=gpurun_out; mkdir -p $OUT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:metrics_select -c 1 -o $OUT/select_full -f \
  python tools/metrics_timing.py 4 > $OUT/ncu_select.log 2>&1
echo "rc=$?" >> $OUT/ncu_select.log
