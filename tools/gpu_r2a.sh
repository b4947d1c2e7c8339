#!/bin/bash
# Round-2 baseline: GPU tests, config 4 / 3 / shard-size benches (device value only).
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r2a}
nvidia-smi > $OUT/smi_$TAG.txt 2>&1; lscpu > $OUT/lscpu_$TAG.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 600 -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_cfg4_$TAG.log 2>&1
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-e2e --cpu-sample 16 > $OUT/bench_cfg3_$TAG.log 2>&1
for sd in 4 8 16; do timeout 600 python bench.py --seeds $sd --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/bench_cfg4_s${sd}_$TAG.log 2>&1; done
