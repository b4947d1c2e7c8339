# round-2: plan's per-segment sorts on their own threads (e2e phases)
OUT=gpurun_out; mkdir -p $OUT; TAG=r2bh
CACE_TIMING=1 timeout 600 python tools/e2e_timing.py > $OUT/e2e_timing_$TAG.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --e2e-steps 5 --parity-sample 64 --cpu-sample 0 > $OUT/bench_cfg4_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -q -x > $OUT/pytest_plan_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_plan_$TAG.log
