#!/bin/bash
# Round check: GPU tests, smoke, default bench (config 4), config 3, 131k shard, launch list.
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r2d}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu_$TAG.txt
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py smoke > $OUT/smoke_$TAG.log 2>&1; echo "rc=$?" >> $OUT/smoke_$TAG.log
timeout 900 python bench.py > $OUT/bench_cfg4_$TAG.log 2>&1; echo "rc=$?" >> $OUT/bench_cfg4_$TAG.log
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --parity-sample 256 > $OUT/bench_cfg3_$TAG.log 2>&1
timeout 600 python bench.py --seeds 4 --steps 3 --warmup 3 --parity-sample 256 > $OUT/bench_s4_$TAG.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
  --log-file $OUT/launches_cfg4_$TAG.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --parity-sample 0 > /dev/null 2>&1
