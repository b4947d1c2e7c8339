# round-2: arrival-vs-cursor test on clock bit patterns (lane kernels) vs the fp64 compare
OUT=gpurun_out; mkdir -p $OUT; TAG=r2bc
CACE_GPU_LIB=$PWD/_build/arrint.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $OUT/pytest_arrint_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_arrint_$TAG.log
export AB_ARGS="--seeds 32;--seeds 4;--seeds 8;--config 3"
bash tools/gpu_ab_libs.sh arrint_$TAG default _build/arrint.so default _build/arrint.so
