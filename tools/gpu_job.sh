# round-2 last check on the committed library: smoke, default bench line, reference arm
OUT=gpurun_out; mkdir -p $OUT; TAG=r2bk
timeout 300 python __graft_entry__.py smoke > $OUT/smoke_$TAG.log 2>&1; echo "rc=$?" >> $OUT/smoke_$TAG.log
timeout 900 python bench.py > $OUT/bench_cfg4_$TAG.log 2>&1
timeout 900 python bench.py --impl reference > $OUT/bench_reference_$TAG.log 2>&1
