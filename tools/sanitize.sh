#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py (every path, small inputs, oracle-checked).
# usage (GPU box): bash tools/sanitize.sh [outdir]   -> <outdir>/r02_sanitizer_<tool>.log
set -u
out=${1:-gpurun_out}
mkdir -p "$out"
cs=/usr/local/cuda/bin/compute-sanitizer
rc=0
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  [ "$tool" = initcheck ] && extra="--track-unused-memory no"
  timeout 1500 $cs --tool $tool $extra --error-exitcode 9 --kernel-name regex:'k_' \
      python tools/sanitize_cases.py > "$out/r02_sanitizer_$tool.log" 2>&1
  r=$?
  echo "$tool exit $r" | tee -a "$out/r02_sanitizer_summary.txt"
  tail -3 "$out/r02_sanitizer_$tool.log" >> "$out/r02_sanitizer_summary.txt"
  [ $r -ne 0 ] && rc=$r
done
exit $rc
