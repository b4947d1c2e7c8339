#!/bin/bash
OUT=gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py > $OUT/sanitize_$tool.log 2>&1
  echo "rc=$?" >> $OUT/sanitize_$tool.log
done
