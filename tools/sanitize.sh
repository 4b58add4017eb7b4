#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py (memcheck, racecheck, synccheck)
for t in memcheck racecheck synccheck; do
  compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t exit=$?" >> gpurun_out/sanitize_summary.txt
  tail -4 gpurun_out/sanitize_$t.log >> gpurun_out/sanitize_summary.txt
done
