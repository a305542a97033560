#!/bin/bash
# compute-sanitizer over the sanitize_run.py cases; logs in gpurun_out/san_<tool>_<case>.log
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  for c in c1_step crowded c3_render det; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 100 python scripts/sanitize_run.py $c \
      > gpurun_out/san_${tool}_${c}.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_${c}.log | tail -1)"
  done
done
