#!/bin/bash
# RunMetrics warm timing vs sample budget (config 4, 32 seeds).
OUT=gpurun_out; mkdir -p $OUT; L=$OUT/metrics_budget.log; : > $L
for b in 60000 100000 140000; do
  echo "== budget $b MB" >> $L
  CACE_METRICS_BUDGET_MB=$b timeout 600 python tools/metrics_timing.py 32 2>&1 | grep run_metrics >> $L
done
echo "== default" >> $L
timeout 600 python tools/metrics_timing.py 32 2>&1 | grep run_metrics >> $L
