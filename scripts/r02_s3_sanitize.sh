#!/bin/bash
# compute-sanitizer over the one-pass kernels: the harness at a capped grid (several
# tiles per CTA: deferred scatter, stage reuse, look-back across CTAs, ragged tail),
# then every libms kernel through scripts/sanitize_cases.py
mkdir -p gpurun_out/r02s3
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02s3
for tool in memcheck racecheck synccheck; do
  for args in "0 0 1 4 100000" "0 1 1 4 70001"; do
    echo "== $tool koh $args" >> $O/sanitize_ko_$tool.txt
    timeout 900 compute-sanitizer --tool $tool bin/koh_san $args >> $O/sanitize_ko_$tool.txt 2>&1; echo "rc=$?" >> $O/sanitize_ko_$tool.txt
  done
  timeout 1500 compute-sanitizer --tool $tool python scripts/sanitize_cases.py > $O/sanitize_$tool.txt 2>&1; echo "rc=$?" >> $O/sanitize_$tool.txt
done
