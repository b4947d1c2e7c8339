#!/bin/bash
# Round-style check: GPU tests, smoke, default bench (config 4), reference arm,
# config-5 calibration, ncu launch list of the default bench.
TAG=${1:-round}
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 600 > $OUT/pytest_gpu_$TAG.log 2>&1
echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1
echo "rc=$?" >> $OUT/smoke_$TAG.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > $OUT/clocks_$TAG.csv &
SMI=$!
timeout 1200 python bench.py > $OUT/bench_$TAG.log 2>&1
echo "rc=$?" >> $OUT/bench_$TAG.log
kill $SMI
timeout 600 python bench.py --impl reference > $OUT/bench_ref_$TAG.log 2>&1
echo "rc=$?" >> $OUT/bench_ref_$TAG.log
timeout 900 python bench.py --config 5 --requests ${CFG5_N:-1000000} --scenarios ${CFG5_S:-2048} --steps 2 --warmup 1 --e2e-steps 1 --cpu-sample 4 > $OUT/bench_cfg5_$TAG.log 2>&1
echo "rc=$?" >> $OUT/bench_cfg5_$TAG.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
echo "rc=$?" >> $OUT/ncu_launch_$TAG.log
