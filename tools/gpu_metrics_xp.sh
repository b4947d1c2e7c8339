#!/bin/bash
# RunMetrics pipeline knobs (exp/mx.so): select off, sample stores off.
OUT=gpurun_out; mkdir -p $OUT; L=$OUT/metrics_xp.log; : > $L
run() { echo "== $*" >> $L; env CACE_GPU_LIB=exp/mx.so CACE_TIMING=1 "$@" timeout 600 python tools/metrics_timing.py 32 2>&1 | grep -E "replay\+select|run_metrics" >> $L; }
run CACE_XP_NOSELECT=1
run CACE_XP_NOSELECT=1 CACE_XP_NOSTORE=1
