#!/bin/bash
# ncu --set full of kernels: SPECS="regex:workload:m:out ..."; exports text summaries, drops big reports
mkdir -p gpurun_out/r02
export PATH=/usr/local/cuda/bin:$PATH
for spec in $SPECS; do
  IFS=: read -r K W M OUT <<< "$spec"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
     -o /tmp/$OUT -f python scripts/prof_driver.py --workload $W --m $M > gpurun_out/r02/ncu_$OUT.log 2>&1
  ncu -i /tmp/$OUT.ncu-rep --page details > gpurun_out/r02/${OUT}_details.txt 2>&1
  ncu -i /tmp/$OUT.ncu-rep --page raw --csv > gpurun_out/r02/${OUT}_raw.csv 2>&1
  ncu -i /tmp/$OUT.ncu-rep --page source --csv > /tmp/${OUT}_source.csv 2>&1
  gzip -c /tmp/${OUT}_source.csv > gpurun_out/r02/${OUT}_source.csv.gz
done
