#!/bin/bash
# ncu --set full of the RunMetrics pipeline's kernels (config 4, 4 seeds):
# one samples-only replay launch (C=6) and one select launch.
OUT=gpurun_out; mkdir -p $OUT
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:replay_lane_kernel -c 1 -o $OUT/metrics_replay_full -f \
  python tools/metrics_timing.py 4 > $OUT/ncu_mrep.log 2>&1
echo "rc=$?" >> $OUT/ncu_mrep.log
[ -n "$SKIP_SELECT" ] || timeout 900 ncu --set full --import-source on --clock-control none -k regex:metrics_select -c 1 -o $OUT/metrics_select_full -f \
  python tools/metrics_timing.py 4 > $OUT/ncu_msel.log 2>&1
echo "rc=$?" >> $OUT/ncu_msel.log
