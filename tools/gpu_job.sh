# round-2: verify the current library (wide-mode window load) -- tests, config 5 full, cfg3 check.
OUT=gpurun_out; mkdir -p $OUT; TAG=r2an
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 1500 python bench.py --config 5 --steps 2 --warmup 3 --e2e-steps 1 --parity-sample 16 --cpu-sample 8 > $OUT/bench_cfg5_$TAG.log 2>&1
AB_ARGS="--seeds 32;--config 3" bash tools/gpu_ab_env.sh ${TAG} ""
