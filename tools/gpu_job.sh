# round-2: exact-fallback pruning only in the rolled per-capacity instantiations.
OUT=gpurun_out; mkdir -p $OUT; TAG=r2ae
AB_ARGS="--seeds 32;--seeds 16;--seeds 8;--seeds 4;--config 3" bash tools/gpu_ab_libs.sh ${TAG} default _variants/libcace_base.so
