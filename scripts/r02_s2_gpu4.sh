#!/bin/bash
mkdir -p gpurun_out/r02s2
O=gpurun_out/r02s2
timeout 1200 python -m pytest tests/test_gpu_sssp.py -q -p no:cacheprovider -x > $O/gpu4_sssp.txt 2>&1; echo "rc=$?" >> $O/gpu4_sssp.txt
: > $O/gpu4_bench.txt
for wm in ms_keys_spl:32 ms_keys_spl:256 ms_pairs_spl:256 ms_keys_large:1024 ms_keys_large:4096 ms_keys_large:65536 ms_pairs_large:4096 sssp_rmat:10; do
  IFS=: read -r W M <<< "$wm"
  timeout 600 python bench.py --workload $W --m $M --steps 10 --warmup 3 --no-sweep >> $O/gpu4_bench.txt 2>> $O/gpu4_bench.err
done
