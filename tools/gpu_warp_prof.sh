#!/bin/bash
OUT=gpurun_out
TAG=${1:-w}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_warp_kernel -c 1 -o $OUT/prof_warp_$TAG \
  python bench.py --config 5 --requests 200000 --scenarios 2048 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ncu_warp_$TAG.log 2>&1
echo "rc=$?" >> $OUT/ncu_warp_$TAG.log
CACE_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 \
  bench.py --gpus 2 --requests 20000 --seeds 4 --steps 2 --warmup 1 --e2e-steps 1 > $OUT/bench_2rank_$TAG.log 2>&1
echo "rc=$?" >> $OUT/bench_2rank_$TAG.log
