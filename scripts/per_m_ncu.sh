#!/bin/bash
# per-m ncu table: the prescan and postscan kernels of one multisplit, m = 2..256, keys and pairs
mkdir -p gpurun_out/r02s2/perm
export PATH=/usr/local/cuda/bin:$PATH
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_requests_srcunit_tex_op_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"
for w in ms_keys ms_pairs; do
  for m in 2 4 8 16 32 64 128 256; do
    timeout 300 ncu --metrics $M --clock-control none -k regex:"km_|kf_meta|kr_" --csv \
      python scripts/prof_driver.py --workload $w --m $m --reps 2 > gpurun_out/r02s2/perm/${w}_m${m}.csv 2>/dev/null
  done
done
timeout 300 ncu --metrics $M --clock-control none -k regex:"km_|kf_meta|kr_" --csv \
  python scripts/prof_driver.py --workload ms_pairs_c3 --m 256 --reps 2 > gpurun_out/r02s2/perm/ms_pairs_c3_m256.csv 2>/dev/null
