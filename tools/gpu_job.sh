# round-2: racecheck after the wide-mode single-writer fix, tests, default bench, config 5 full,
# launch lists (traffic) for config 4, config 3 and the shards.
OUT=gpurun_out; mkdir -p $OUT; TAG=r2k
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_run.py > $OUT/sanitize_racecheck_$TAG.log 2>&1; echo "rc=$?" >> $OUT/sanitize_racecheck_$TAG.log
timeout 1500 python -m pytest tests -m gpu -x -q -rf --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 900 python bench.py > $OUT/bench_cfg4_$TAG.log 2>&1
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --parity-sample 256 > $OUT/bench_cfg3_$TAG.log 2>&1
timeout 1500 python bench.py --config 5 --steps 2 --warmup 3 --e2e-steps 1 --parity-sample 16 --cpu-sample 8 > $OUT/bench_cfg5_$TAG.log 2>&1
for a in "--seeds 32" "--seeds 4" "--config 3"; do t=$(echo $a | tr -d ' -')
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
    --log-file $OUT/launches_${t}_$TAG.csv python bench.py $a --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
