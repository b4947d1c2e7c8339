# round-2 final evidence (exact-tie build): default bench, reference arm, shards, config 3, metrics, launch list.
OUT=gpurun_out; mkdir -p $OUT; TAG=r2aj
timeout 300 python __graft_entry__.py smoke > $OUT/smoke_$TAG.log 2>&1; echo "rc=$?" >> $OUT/smoke_$TAG.log
timeout 900 python bench.py > $OUT/bench_cfg4_$TAG.log 2>&1
timeout 900 python bench.py --impl reference > $OUT/bench_reference_$TAG.log 2>&1
for s in 16 8 4; do timeout 900 python bench.py --seeds $s --steps 5 --warmup 3 --parity-sample 256 --cpu-sample 32 > $OUT/bench_s${s}_$TAG.log 2>&1; done
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --parity-sample 256 > $OUT/bench_cfg3_$TAG.log 2>&1
timeout 900 python bench.py --config 2 --steps 5 --warmup 3 --parity-sample 2 > $OUT/bench_cfg2_$TAG.log 2>&1
timeout 1200 python bench.py --metrics --steps 2 --warmup 1 --parity-sample 32 > $OUT/bench_metrics_cfg4_$TAG.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file $OUT/launches_seeds32_$TAG.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
