#!/bin/bash
# One gpurun pass: GPU parity tests, smoke, a calibration bench, ncu launch list + one full capture.
# Usage (from repo root, on the GPU box): bash tools/gpu_check.sh [tag]
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi -L > $OUT/gpu_$TAG.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)|Flags" | cut -c1-300 >> $OUT/gpu_$TAG.txt
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 600 > $OUT/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1
echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 600 python bench.py --requests 20000 --seeds 4 --steps 3 --warmup 3 --e2e-steps 1 --cpu-sample 8 > $OUT/bench_small_$TAG.log 2>&1
echo "bench rc=$?" >> $OUT/bench_small_$TAG.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --requests 20000 --seeds 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
echo "ncu launches rc=$?" >> $OUT/ncu_launch_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:replay_lane_kernel -s 3 -c 1 -o $OUT/prof_$TAG \
  python bench.py --requests 20000 --seeds 4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?" >> $OUT/ncu_full_$TAG.log
