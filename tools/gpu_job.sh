# round-2: ncu --set full of the mixed-capacity (runtime-capacity) launch on the 131k shard
OUT=gpurun_out; mkdir -p $OUT; TAG=r2aw
bash tools/gpu_ncu.sh ${TAG}_mixed 'replay_lane_kernel.*true' --seeds 4
