#!/bin/bash
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests/test_gpu_onesweep.py tests/test_gpu_sharded.py tests/test_gpu_repeat.py tests/test_gpu_fullsize.py -q -p no:cacheprovider > gpurun_out/os_pytest.txt 2>&1; echo "pytest exit $?" >> gpurun_out/os_pytest.txt
for w in "sort_keys" "sort_pairs" "ms_pairs_os --m 256" "ms_keys_os --m 256"; do
  echo "== $w" >> gpurun_out/os_bench.txt
  timeout 300 python bench.py --no-cpu-baseline --no-sweep --steps 10 --warmup 3 --workload $w >> gpurun_out/os_bench.txt 2>> gpurun_out/os_bench.err
done
