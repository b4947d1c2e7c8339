# round-2: multi-device entry finds the first failing scenario while scattering back; GPU tests
OUT=gpurun_out; mkdir -p $OUT; TAG=r2bi
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 900 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu_$TAG.log
