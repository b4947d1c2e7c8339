# round-2: event-cursor idleness test as one integer borrow chain (sckey) vs fp64 compares
OUT=gpurun_out; mkdir -p $OUT; TAG=r2ay
CACE_GPU_LIB=$PWD/_build/sckey.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $OUT/pytest_sckey_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_sckey_$TAG.log
export AB_ARGS="--seeds 32;--seeds 4;--seeds 8;--config 3"
bash tools/gpu_ab_libs.sh sckey_$TAG default _build/sckey.so default _build/sckey.so
