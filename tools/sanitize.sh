#!/bin/bash
# compute-sanitizer over tests/sanitize_smoke.py (small shapes), on the box:
#   gpurun -- bash tools/sanitize.sh
# Round 2: the GPU pool refuses compute-sanitizer ("closed on this pool":
# runs under it have left GPUs needing a reset); the attempt and its message
# are kept in profiles/r02_sanitizer_closed.txt.
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  SANITIZE_SMALL=1 timeout 900 $CS --tool $tool --print-limit 20 python tests/sanitize_smoke.py \
      > gpurun_out/sanitize/$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize/summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Invalid|Error" gpurun_out/sanitize/$tool.txt | tail -5 >> gpurun_out/sanitize/summary.txt
done
