OUT=gpurun_out; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q -rf --timeout 900 > $OUT/pytest_gpu_r2i.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_r2i.log
bash tools/gpu_ab_env.sh r2i "" "CACE_PERSIST=0" "CACE_LATENCY_WAVES=0"
bash tools/gpu_ncu.sh r2i_cfg5w "replay_lane_wide_kernel" --config 5 --requests 200000 --parity-sample 0
