#!/bin/bash
# Config 5 (256 models, capacity 32, window 1024): pool tests, then the wide lane kernel vs the warp kernel.
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-c5}; N=${CFG5_N:-1000000}
timeout 900 python -m pytest tests/test_gpu_pools.py tests/test_gpu_warp_kernel.py tests/test_gpu_parity.py -q -x > $OUT/pytest_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_$TAG.log
for k in auto warp; do
  timeout 1200 python bench.py --config 5 --requests $N --steps 2 --warmup 1 --e2e-steps 1 --parity-sample 16 --cpu-sample 4 --kernel $k > $OUT/bench_cfg5_${k}_$TAG.log 2>&1
done
