#!/bin/bash
# DRAM bytes of KF for several (workload, m): write/read amplification vs bucket run length
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
for cfg in ${CFGS:-"ms_keys 256" "ms_keys 128" "ms_keys 64" "ms_keys 8"}; do
  set -- $cfg
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed \
     --clock-control none -k regex:kf_fused -s 2 -c 1 --csv \
     python scripts/prof_driver.py --workload $1 --m $2 > gpurun_out/dram_$1_$2.csv 2>&1
done
