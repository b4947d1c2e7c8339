#!/bin/bash
# GPU tests, default bench (strong, N=1, parity sample 1024), 2-rank gloo bench, config 3.
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-r2c}
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.log 2>&1; echo "rc=$?" >> $OUT/bench_$TAG.log
CACE_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 2 --seeds 4 --steps 2 --warmup 3 --e2e-steps 1 \
    > $OUT/bench_2rank_$TAG.log 2>&1; echo "rc=$?" >> $OUT/bench_2rank_$TAG.log
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --parity-sample 256 > $OUT/bench_cfg3_$TAG.log 2>&1
