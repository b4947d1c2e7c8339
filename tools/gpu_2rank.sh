#!/bin/bash
# Two ranks sharing one GPU over gloo: the N>1 bench flow (weak and strong).
OUT=gpurun_out
mkdir -p $OUT
for mode in weak strong; do
  CACE_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29555 \
    bench.py --gpus 2 --requests 20000 --seeds 4 --steps 2 --warmup 3 --e2e-steps 1 --scaling $mode \
    > $OUT/bench_2rank_$mode.log 2>&1
  echo "rc=$?" >> $OUT/bench_2rank_$mode.log
done
