#!/bin/bash
mkdir -p gpurun_out/r02s2
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02s2
for spec in kf_meta_wide:ms_pairs_c3:256:p4_kfw_pairs256; do
  IFS=: read -r K W M OUT <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
     -o /tmp/$OUT -f python scripts/prof_driver.py --workload $W --m $M > $O/ncu_$OUT.log 2>&1
  python scripts/ncu_summary.py /tmp/$OUT.ncu-rep > $O/${OUT}_summary.txt 2>&1
  python scripts/sass_stalls.py /tmp/$OUT.ncu-rep > $O/${OUT}_stalls.txt 2>&1
  ncu -i /tmp/$OUT.ncu-rep --page raw --csv > $O/${OUT}_raw.csv 2>&1
done
