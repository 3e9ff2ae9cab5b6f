#!/bin/bash
# round 2 session 3: first GPU check of the one-pass pipeline (f1)
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python -m pytest tests/test_gpu_onesweep.py -q -x -p no:cacheprovider > gpurun_out/os_pytest.txt 2>&1; echo "pytest exit $?" >> gpurun_out/os_pytest.txt
for w in "sort_keys" "sort_pairs" "sort_keys_passes" "sort_pairs_passes" "ms_keys_os --m 32" "ms_keys_os --m 256" "ms_pairs_os --m 256" "ms_keys --m 256"; do
  echo "== $w" >> gpurun_out/os_bench.txt
  timeout 300 python bench.py --no-cpu-baseline --no-sweep --steps 10 --warmup 3 --workload $w >> gpurun_out/os_bench.txt 2>> gpurun_out/os_bench.err
done
