#!/bin/bash
# Sanitizers + first-call (cold process) RunMetrics timing vs sample budget.
OUT=gpurun_out; mkdir -p $OUT
bash tools/gpu_sanitize.sh
CACE_TIMING=1 timeout 600 python tools/metrics_timing.py 32 > $OUT/cold_default.log 2>&1
CACE_METRICS_BUDGET_MB=30000 CACE_TIMING=1 timeout 600 python tools/metrics_timing.py 32 > $OUT/cold_30g.log 2>&1
