#!/bin/bash
# round 2, call 1: GPU tests, compute-sanitizer over every kernel, a bench line
mkdir -p gpurun_out/r02
export PATH=/usr/local/cuda/bin:$PATH
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02/gpu1_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02/gpu1_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/gpu1_pytest.txt
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_cases.py \
    > gpurun_out/r02/sanitize_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/r02/sanitize_$tool.txt
done
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/gpu1_bench.json 2> gpurun_out/r02/gpu1_bench.err
