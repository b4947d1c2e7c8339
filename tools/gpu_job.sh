# round-2: parallel plan (sort / order phases) -- tests, e2e phases, default bench.
OUT=gpurun_out; mkdir -p $OUT; TAG=r2au
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
CACE_TIMING=1 timeout 600 python tools/e2e_timing.py > $OUT/e2e_timing_$TAG.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --e2e-steps 4 --parity-sample 64 --cpu-sample 16 > $OUT/bench_cfg4_$TAG.log 2>&1
