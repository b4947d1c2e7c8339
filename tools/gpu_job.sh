# round-2: compile-time pool size (MC) for the RunMetrics sample kernels and the config-5 wide kernel.
OUT=gpurun_out; mkdir -p $OUT; TAG=r2r
timeout 900 python -m pytest tests/test_gpu_metrics.py tests/test_gpu_pools.py tests/test_gpu_warp_kernel.py -x -q > $OUT/pytest_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_$TAG.log
AB_ARGS="--config 5 --requests 1000000" bash tools/gpu_ab_libs.sh ${TAG} default _variants/libcace_nomc.so
for lib in default _variants/libcace_nomc.so; do L=""; [ "$lib" != "default" ] && L="CACE_GPU_LIB=$PWD/$lib"
  env $L timeout 900 python bench.py --metrics --steps 2 --warmup 1 --parity-sample 8 2>&1 | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'metrics_cfg4', round(d['value']/1e9,2), round(d['ms_per_step'],1), d['parity_sample'])" >> $OUT/ab_$TAG.txt
done
