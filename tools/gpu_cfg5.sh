#!/bin/bash
# BASELINE config 5 at full size (8192 scenarios x 10M-request bursty trace, 256 CodeLLMs, capacity 32,
# window 1024) with a 16-scenario port-checked parity sample, then an ncu --set full capture of the
# wide-pool lane kernel on a 1M-request slice.  Usage: bash tools/gpu_cfg5_r2.sh TAG
TAG=${1:-r2}
OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python bench.py --config 5 --steps 2 --warmup 3 --e2e-steps 1 --parity-sample 16 --cpu-sample 8 \
  > $OUT/bench_cfg5_$TAG.log 2>&1; echo "rc=$?" >> $OUT/bench_cfg5_$TAG.log
bash tools/gpu_ncu.sh ${TAG}_cfg5w "replay_lane_wide_kernel" --config 5 --requests 200000 --parity-sample 0
