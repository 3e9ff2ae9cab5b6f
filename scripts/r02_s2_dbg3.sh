#!/bin/bash
mkdir -p gpurun_out/r02s2
O=gpurun_out/r02s2/dbg3.txt; : > $O
for args in "fresh 16777216 256 1" "keep 16777216 256 1" "sync 16777216 256 1" "zero 16777216 256 1" "fresh 16777216 256 0" "fresh 16777216 64 0" "fresh 1048576 256 1"; do
  echo "== $args" >> $O
  timeout 300 python scripts/dbg_r02s2c.py $args >> $O 2>&1
done
echo "== launch blocking" >> $O
CUDA_LAUNCH_BLOCKING=1 timeout 300 python scripts/dbg_r02s2c.py fresh 16777216 256 1 >> $O 2>&1
