#!/bin/bash
# launch list of the default bench command + ncu --set full of the large-m kernels and kf_meta m=4/32
mkdir -p gpurun_out/r02s2
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02s2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu-baseline > $O/launches_default.csv 2> $O/launches_default.err
for spec in kf_meta_wide:ms_keys:256:kfw_keys256 kf_meta_wide:ms_pairs_c3:256:kfw_pairs256 km_meta_wide:ms_keys:256:kmw_keys256 \
            kf_meta:ms_keys:4:kfm_keys4 kf_meta:ms_keys:32:kfm_keys32 km_tile_meta:ms_keys:4:km_keys4; do
  IFS=: read -r K W M OUT <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
     -o /tmp/$OUT -f python scripts/prof_driver.py --workload $W --m $M > $O/ncu_$OUT.log 2>&1
  python scripts/ncu_summary.py /tmp/$OUT.ncu-rep > $O/${OUT}_summary.txt 2>&1
  python scripts/sass_stalls.py /tmp/$OUT.ncu-rep > $O/${OUT}_stalls.txt 2>&1
  ncu -i /tmp/$OUT.ncu-rep --page raw --csv > $O/${OUT}_raw.csv 2>&1
done
