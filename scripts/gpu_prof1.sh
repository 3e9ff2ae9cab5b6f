#!/bin/bash
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
# strategy variants (evidence for the per-m choice)
for v in "MS_HIST=match MS_RANK=match" "MS_HIST=atomic MS_RANK=peers"; do
  env $v timeout 600 python bench.py --no-cpu-baseline --steps 10 > "gpurun_out/bench_${v// /_}.json" 2>>gpurun_out/variants.err
done
# launch list of the default bench command (cold-cache, serialised)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --no-sweep --no-cpu-baseline --steps 3 --warmup 3 > /dev/null 2>gpurun_out/launches.err
# full sets for the postscan and prescan at m=32 keys, and postscan keys m=2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ks_postscan -s 2 -c 1 \
   -o gpurun_out/ks_keys_m32 python scripts/prof_driver.py --workload ms_keys --m 32 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kh_prescan -s 2 -c 1 \
   -o gpurun_out/kh_keys_m32 python scripts/prof_driver.py --workload ms_keys --m 32 > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ks_postscan -s 2 -c 1 \
   -o gpurun_out/ks_keys_m2 python scripts/prof_driver.py --workload ms_keys --m 2 > gpurun_out/ncu3.log 2>&1
