#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py: memcheck / racecheck / synccheck with the
# host-driven level loop, memcheck with the default device loop (CUDA graph)
rm -f gpurun_out/sanitize_summary.txt
for t in memcheck racecheck synccheck; do
  compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/sanitize_$t.log 2>&1
  echo "$t (host loop) exit=$?" >> gpurun_out/sanitize_summary.txt
  grep -E "SUMMARY|sanitize run ok" gpurun_out/sanitize_$t.log >> gpurun_out/sanitize_summary.txt
done
compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_run.py --graph > gpurun_out/sanitize_memcheck_graph.log 2>&1
echo "memcheck (device loop) exit=$?" >> gpurun_out/sanitize_summary.txt
grep -E "SUMMARY|sanitize run ok" gpurun_out/sanitize_memcheck_graph.log >> gpurun_out/sanitize_summary.txt
