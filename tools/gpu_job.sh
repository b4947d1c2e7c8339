# round-2: mixed-capacity launch up to 1.8 waves; shard lines + tests + smoke on the final library
OUT=gpurun_out; mkdir -p $OUT; TAG=r2bq
timeout 900 python bench.py --seeds 5 --steps 5 --warmup 3 --parity-sample 256 --cpu-sample 0 > $OUT/bench_s5_$TAG.log 2>&1
timeout 900 python bench.py --seeds 4 --steps 5 --warmup 3 --parity-sample 256 --cpu-sample 32 > $OUT/bench_s4_$TAG.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py smoke > $OUT/smoke_$TAG.log 2>&1; echo "rc=$?" >> $OUT/smoke_$TAG.log
timeout 900 python bench.py > $OUT/bench_cfg4_$TAG.log 2>&1
