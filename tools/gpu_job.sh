# round-2 final verification of the committed library (all bench lines, smoke, sanitizers)
OUT=gpurun_out; mkdir -p $OUT; TAG=r2bg
timeout 300 python __graft_entry__.py smoke > $OUT/smoke_$TAG.log 2>&1; echo "rc=$?" >> $OUT/smoke_$TAG.log
for t in racecheck memcheck synccheck initcheck; do timeout 1200 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_run.py > $OUT/sanitize_${t}_$TAG.log 2>&1; echo "rc=$?" >> $OUT/sanitize_${t}_$TAG.log; done
timeout 900 python bench.py > $OUT/bench_cfg4_$TAG.log 2>&1
timeout 900 python bench.py --impl reference > $OUT/bench_reference_$TAG.log 2>&1
for s in 16 8 4; do timeout 900 python bench.py --seeds $s --steps 5 --warmup 3 --parity-sample 256 --cpu-sample 32 > $OUT/bench_s${s}_$TAG.log 2>&1; done
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --parity-sample 256 > $OUT/bench_cfg3_$TAG.log 2>&1
timeout 900 python bench.py --config 2 --steps 5 --warmup 3 > $OUT/bench_cfg2_$TAG.log 2>&1
timeout 1500 python bench.py --config 5 --steps 2 --warmup 3 --e2e-steps 1 --parity-sample 16 --cpu-sample 8 > $OUT/bench_cfg5_$TAG.log 2>&1
timeout 1200 python bench.py --metrics --steps 2 --warmup 1 --parity-sample 32 > $OUT/bench_metrics_cfg4_$TAG.log 2>&1
