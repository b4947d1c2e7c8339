#!/bin/bash
# RunMetrics per-chunk device timeline (CACE_TIMING), config 4 32 seeds; knob CACE_XP_LAT.
OUT=gpurun_out; mkdir -p $OUT
CACE_TIMING=1 timeout 600 python tools/metrics_timing.py 32 > $OUT/metrics_tl.log 2>&1
CACE_XP_LAT=0 CACE_TIMING=1 timeout 600 python tools/metrics_timing.py 32 > $OUT/metrics_tl_lat0.log 2>&1
timeout 600 python tools/metrics_timing.py 4 > $OUT/metrics_tl4.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_conn.log 2>&1
