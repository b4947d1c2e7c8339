# round-2: shallow-sweep policy (mixed launch at MINB 4 below 1.5 waves) on the default library; tests.
OUT=gpurun_out; mkdir -p $OUT; TAG=r2z
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
for s in 32 16 8 4; do timeout 900 python bench.py --seeds $s --steps 5 --warmup 3 --parity-sample 256 --cpu-sample 32 > $OUT/bench_s${s}_$TAG.log 2>&1; done
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --parity-sample 256 > $OUT/bench_cfg3_$TAG.log 2>&1
AB_ARGS="--seeds 4;--seeds 2;--seeds 1" bash tools/gpu_ab_env.sh ${TAG} "" "CACE_MIXED=0"
