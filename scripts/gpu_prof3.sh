#!/bin/bash
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
W=${WL:-ms_keys}; M=${MM:-32}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kf_fused -s 2 -c 1 \
   -o gpurun_out/kf_${W}_m${M} python scripts/prof_driver.py --workload $W --m $M > gpurun_out/ncu_${W}_${M}.log 2>&1
if [ -n "$MM2" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kf_fused -s 2 -c 1 \
   -o gpurun_out/kf_${W}_m${MM2} python scripts/prof_driver.py --workload $W --m $MM2 > gpurun_out/ncu_${W}_${MM2}.log 2>&1
fi
