# round-2: occupancy tiers by sweep depth (MINB 3 / 4 / 5) on the in-tree library.
OUT=gpurun_out; mkdir -p $OUT; TAG=r2n
timeout 1500 python -m pytest tests -m gpu -x -q -rf --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
AB_ARGS="--seeds 32;--seeds 16;--seeds 8;--seeds 4;--config 3" bash tools/gpu_ab_env.sh ${TAG}_tiers "" "CACE_LANE_MINB=5"
