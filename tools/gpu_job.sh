# round-2: p1 shared by exact candidates with equal last_used.
OUT=gpurun_out; mkdir -p $OUT; TAG=r2af
AB_ARGS="--seeds 32;--seeds 8;--seeds 4;--config 3" bash tools/gpu_ab_libs.sh ${TAG} default _variants/libcace_base.so default _variants/libcace_base.so
