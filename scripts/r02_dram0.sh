#!/bin/bash
# round-2 baseline: DRAM bytes + time of kf_fused at large m (default vs carry), current build
mkdir -p gpurun_out/r02
export PATH=/usr/local/cuda/bin:$PATH
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__average_warp_latency_issue_stalled_mio_throttle.ratio"
run() { # tag env workload m
  tag=$1; shift; envs=$1; shift
  env $envs timeout 300 ncu --metrics $M --clock-control none -k regex:kf_fused -s 2 -c 1 --csv \
     python scripts/prof_driver.py --workload $1 --m $2 > gpurun_out/r02/dram0_${tag}.csv 2>&1
}
run pairs_c3_256 "X=1" ms_pairs_c3 256
run pairs_c3_256_carry "MS_CARRY=1" ms_pairs_c3 256
run keys_256 "X=1" ms_keys 256
run keys_256_carry "MS_CARRY=1" ms_keys 256
run keys_256_noinc "MS_NO_RANK_INC=1" ms_keys 256
run keys_64 "X=1" ms_keys 64
run pairs_256 "X=1" ms_pairs 256
