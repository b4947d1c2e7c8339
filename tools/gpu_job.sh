# round-2: parity file incl. the signed-zero and extreme-magnitude clock tests on the final library
OUT=gpurun_out; mkdir -p $OUT; TAG=r2bd
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf > $OUT/pytest_parity_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_parity_$TAG.log
