#!/bin/bash
# parity + A/B bench lines: default vs env variants ($VARIANTS, ';'-separated env assignments)
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
fi
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for wl in ${WLS:-"ms_keys:32"}; do
  IFS=: read -r W M <<< "$wl"
  for v in "" "${VS[@]}"; do
    tag=$(echo "$W.$M.$v" | tr ' =' '_-')
    env $v timeout 300 python bench.py --no-sweep --no-cpu-baseline --workload $W --m $M --steps 20 > gpurun_out/ab_$tag.json 2>gpurun_out/ab_$tag.err
  done
done
