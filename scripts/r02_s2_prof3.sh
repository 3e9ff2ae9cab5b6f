#!/bin/bash
mkdir -p gpurun_out/r02s2
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02s2
for spec in kf_meta_wide:ms_keys:256:p3_kfw_keys256 km_meta_wide:ms_keys:256:p3_kmw_keys256 kf_meta:ms_keys:32:p3_kfm_keys32 km_tile_meta:ms_keys:32:p3_km_keys32; do
  IFS=: read -r K W M OUT <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
     -o /tmp/$OUT -f python scripts/prof_driver.py --workload $W --m $M > $O/ncu_$OUT.log 2>&1
  python scripts/ncu_summary.py /tmp/$OUT.ncu-rep > $O/${OUT}_summary.txt 2>&1
  python scripts/sass_stalls.py /tmp/$OUT.ncu-rep > $O/${OUT}_stalls.txt 2>&1
done
