#!/bin/bash
# ncu --set full of the one-pass kernels (KO keys / pairs m = 256, KOH of the sort)
mkdir -p gpurun_out/r02s3
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02s3
for spec in ${SPECS:-ko_onesweep:ms_keys_os:256:ko_keys256 ko_onesweep:ms_pairs_os:256:ko_pairs256 ko_hist:sort_keys:256:koh_sort}; do
  IFS=: read -r K W M OUT <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
     -o /tmp/$OUT -f python scripts/prof_driver.py --workload $W --m $M > $O/ncu_$OUT.log 2>&1
  python scripts/ncu_summary.py /tmp/$OUT.ncu-rep $N > $O/${OUT}_summary.txt 2>&1
  python scripts/sass_stalls.py /tmp/$OUT.ncu-rep > $O/${OUT}_stalls.txt 2>&1
  python scripts/src_stalls.py /tmp/$OUT.ncu-rep 50 > $O/${OUT}_src.txt 2>&1
  ncu -i /tmp/$OUT.ncu-rep --page raw --csv > $O/${OUT}_raw.csv 2>&1

done
