#!/bin/bash
mkdir -p gpurun_out/r02s2
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02s2
bash scripts/per_m_ncu.sh
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_cases.py > $O/sanitize_$tool.txt 2>&1
  echo "rc=$?" >> $O/sanitize_$tool.txt
done
