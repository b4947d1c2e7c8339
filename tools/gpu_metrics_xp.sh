#!/bin/bash
# RunMetrics knobs: replay-only (select off) for two builds.
OUT=gpurun_out; mkdir -p $OUT; L=$OUT/metrics_xp.log; : > $L
run() { echo "== $*" >> $L; env CACE_TIMING=1 "$@" timeout 600 python tools/metrics_timing.py 32 2>&1 | grep -E "replay\+select|run_metrics" >> $L; }
run CACE_GPU_LIB=exp/mx2.so CACE_XP_NOSELECT=1
run CACE_GPU_LIB=exp/mx2.so
run CACE_GPU_LIB=exp/mx1.so
