# round-2: occupancy tier crossover moved to 2.5 waves; shard bench lines + tests
OUT=gpurun_out; mkdir -p $OUT; TAG=r2bn
for s in 16 8 4; do timeout 900 python bench.py --seeds $s --steps 5 --warmup 3 --parity-sample 256 --cpu-sample 32 > $OUT/bench_s${s}_$TAG.log 2>&1; done
timeout 900 python bench.py --seeds 12 --steps 5 --warmup 3 --parity-sample 256 --cpu-sample 0 > $OUT/bench_s12_$TAG.log 2>&1
timeout 900 python bench.py --seeds 6 --steps 5 --warmup 3 --parity-sample 256 --cpu-sample 0 > $OUT/bench_s6_$TAG.log 2>&1
timeout 900 python bench.py > $OUT/bench_cfg4_$TAG.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
