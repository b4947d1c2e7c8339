# round-2: RunMetrics line (config 4 and config 3) through the public API.
OUT=gpurun_out; mkdir -p $OUT; TAG=r2p
timeout 1200 python bench.py --metrics --steps 2 --warmup 1 --parity-sample 32 > $OUT/bench_metrics_cfg4_$TAG.log 2>&1
timeout 600 python bench.py --metrics --config 3 --steps 3 --warmup 1 --parity-sample 32 > $OUT/bench_metrics_cfg3_$TAG.log 2>&1
