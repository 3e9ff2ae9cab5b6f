#!/bin/bash
# run every bin/koh_* harness binary (scripts/ko_harness.cu variants); ARGS: ';'-separated arg lists
mkdir -p gpurun_out
IFS=';' read -ra LISTS <<< "${ARGS:-25 0;25 1;28 0}"
for b in ${BIN:-bin}/koh_*; do
  for args in "${LISTS[@]}"; do
    echo "== $b $args" >> gpurun_out/ko_runs.txt
    timeout 120 $b $args >> gpurun_out/ko_runs.txt 2>&1
  done
done
