#!/bin/bash
# compute-sanitizer over every libcqs device path (tools/sanitize_cases.py); summaries -> $OUT
OUT=${OUT:-gpurun_out/sanitize}
mkdir -p "$OUT"
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 python tools/sanitize_cases.py \
      > "$OUT/$tool.log" 2>&1
  echo "$tool rc=$?" >> "$OUT/summary.txt"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize cases ok" "$OUT/$tool.log" >> "$OUT/summary.txt"
done
cat "$OUT/summary.txt"
