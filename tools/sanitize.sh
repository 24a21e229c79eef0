#!/bin/bash
# compute-sanitizer over every libcqs device path (tools/sanitize_cases.py); logs + aggregated
# summaries (tools/sanitize_summary.py) -> $OUT
OUT=${OUT:-gpurun_out/sanitize}
mkdir -p "$OUT"
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
CS=/usr/local/cuda/bin/compute-sanitizer
: > "$OUT/summary.txt"
for tool in memcheck racecheck synccheck initcheck; do
  extra="--print-limit 2000"
  [ "$tool" = memcheck ] && extra="$extra --leak-check no"
  [ "$tool" = racecheck ] && extra="--print-limit 20000 --racecheck-report all"
  timeout 1500 $CS --tool $tool $extra python tools/sanitize_cases.py > "$OUT/$tool.log" 2>&1
  echo "== $tool rc=$?" >> "$OUT/summary.txt"
  python tools/sanitize_summary.py "$OUT/$tool.log" >> "$OUT/summary.txt"
  # keep the head of very long logs only
  if [ $(stat -c %s "$OUT/$tool.log") -gt 20000000 ]; then
    head -c 5000000 "$OUT/$tool.log" > "$OUT/$tool.head.log"; rm "$OUT/$tool.log"
  fi
done
cat "$OUT/summary.txt"
