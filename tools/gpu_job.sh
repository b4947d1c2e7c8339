# round-2 final verification (integer cursor key in the lane kernels, fp64 compares in the wide kernel)
OUT=gpurun_out; mkdir -p $OUT; TAG=r2bb
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py smoke > $OUT/smoke_$TAG.log 2>&1; echo "rc=$?" >> $OUT/smoke_$TAG.log
for t in racecheck memcheck; do timeout 1200 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_run.py > $OUT/sanitize_${t}_$TAG.log 2>&1; echo "rc=$?" >> $OUT/sanitize_${t}_$TAG.log; done
timeout 900 python bench.py > $OUT/bench_cfg4_$TAG.log 2>&1
timeout 1500 python bench.py --config 5 --steps 2 --warmup 3 --e2e-steps 1 --parity-sample 16 --cpu-sample 8 > $OUT/bench_cfg5_$TAG.log 2>&1
