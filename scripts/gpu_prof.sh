#!/bin/bash
# ncu --set full of kernels matching $K (regex) for workload $W and m $M -> gpurun_out/$OUT.ncu-rep
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
for spec in $SPECS; do
  IFS=: read -r K W M OUT <<< "$spec"
  timeout 600 ncu --set full --clock-control none -k regex:$K -s 2 -c 1 \
     -o gpurun_out/$OUT python scripts/prof_driver.py --workload $W --m $M > gpurun_out/ncu_$OUT.log 2>&1
done
