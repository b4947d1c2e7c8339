# round-2: mixed-capacity entry list built/uploaded only when replay() chooses the mixed launch (e2e)
OUT=gpurun_out; mkdir -p $OUT; TAG=r2bf
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
CACE_TIMING=1 timeout 600 python tools/e2e_timing.py > $OUT/e2e_timing_$TAG.log 2>&1
timeout 900 python bench.py > $OUT/bench_cfg4_$TAG.log 2>&1
timeout 900 python bench.py --seeds 4 --steps 5 --warmup 3 --parity-sample 256 --cpu-sample 32 > $OUT/bench_s4_$TAG.log 2>&1
