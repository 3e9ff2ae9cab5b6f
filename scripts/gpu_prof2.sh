#!/bin/bash
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kf_fused -s 2 -c 1 \
   -o gpurun_out/kf_keys_m32 python scripts/prof_driver.py --workload ms_keys --m 32 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ku_range -s 2 -c 1 \
   -o gpurun_out/ku_keys_m32 python scripts/prof_driver.py --workload ms_keys --m 32 > gpurun_out/ncu2.log 2>&1
