#!/bin/bash
# compute-sanitizer passes over every kernel layout (tools/sanitize_cfgs.py);
# log in gpurun_out/sanitizer.txt
mkdir -p gpurun_out
: > gpurun_out/sanitizer.txt
for tool in memcheck racecheck synccheck initcheck; do
  echo "== compute-sanitizer --tool $tool" >> gpurun_out/sanitizer.txt
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_cfgs.py >> gpurun_out/sanitizer.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer.txt
done
grep -E "^==|SUMMARY|rc=" gpurun_out/sanitizer.txt
