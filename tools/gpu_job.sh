# round-2: validate the exact-tie shortcut build; ncu of the C = 6 and C = 3 launches.
OUT=gpurun_out; mkdir -p $OUT; TAG=r2ai
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
bash tools/gpu_ncu.sh ${TAG}_C6 "replay_lane_kernel<.int.6," --parity-sample 0
bash tools/gpu_ncu.sh ${TAG}_C3 "replay_lane_kernel<.int.3," --parity-sample 0
