#!/bin/bash
# the whole GPU suite, then launch lists (ncu, cold, serialized) of the sorts
mkdir -p gpurun_out/r02s3
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02s3
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_full.txt 2>&1; echo "pytest exit $?" >> $O/pytest_gpu_full.txt
for w in sort_keys sort_pairs; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
    python scripts/prof_driver.py --workload $w --reps 2 > $O/launches_$w.csv 2> $O/launches_$w.err
done
