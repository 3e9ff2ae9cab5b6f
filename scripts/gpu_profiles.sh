#!/bin/bash
# Round profiles: launch list of the default bench command + ncu --set full of the dominant kernel.
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --no-sweep --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/launches.log 2>&1
for cfg in "ms_keys 32" "ms_keys 2" "ms_pairs 32" "ms_pairs_c3 256"; do
  set -- $cfg
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:kf_fused -s 2 -c 1 \
     -o gpurun_out/kf_$1_m$2 python scripts/prof_driver.py --workload $1 --m $2 > gpurun_out/ncu_$1_$2.log 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:ku_range -s 2 -c 1 \
   -o gpurun_out/ku_ms_keys_m32 python scripts/prof_driver.py --workload ms_keys --m 32 > gpurun_out/ncu_ku.log 2>&1
