# round-2 evidence on the final library: tests, smoke, default bench, reference arm, config 3, shards,
# launch list (traffic), ncu --set full of the C = 6 launch, MINB 3 vs 4 at 131k.
OUT=gpurun_out; mkdir -p $OUT; TAG=r2s
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py smoke > $OUT/smoke_$TAG.log 2>&1; echo "rc=$?" >> $OUT/smoke_$TAG.log
timeout 900 python bench.py > $OUT/bench_cfg4_$TAG.log 2>&1
timeout 900 python bench.py --impl reference > $OUT/bench_reference_$TAG.log 2>&1
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --parity-sample 256 > $OUT/bench_cfg3_$TAG.log 2>&1
for s in 16 8 4; do timeout 900 python bench.py --seeds $s --steps 5 --warmup 3 --parity-sample 256 --cpu-sample 32 > $OUT/bench_s${s}_$TAG.log 2>&1; done
AB_ARGS="--seeds 4;--config 3" bash tools/gpu_ab_env.sh ${TAG}_minb "CACE_LANE_MINB=3" "CACE_LANE_MINB=4"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file $OUT/launches_seeds32_$TAG.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
bash tools/gpu_ncu.sh ${TAG}_C6 "replay_lane_kernel<.int.6," --parity-sample 0
