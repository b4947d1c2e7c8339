# round-2: RunMetrics ring count (chunk size) A/B on config 4.
OUT=gpurun_out; mkdir -p $OUT; TAG=r2ac
for r in 8 4 2; do
  CACE_METRICS_RINGS=$r timeout 900 python bench.py --metrics --steps 2 --warmup 1 --parity-sample 4 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('rings $r', round(d['value']/1e9,2), round(d['ms_per_step'],1), d['parity_sample']['percentiles_bit_exact_mean_1e-12'])" >> $OUT/ab_$TAG.txt
done
CACE_TIMING=1 CACE_METRICS_RINGS=8 timeout 600 python tools/metrics_timing.py 32 > $OUT/metrics_timing_$TAG.log 2>&1
