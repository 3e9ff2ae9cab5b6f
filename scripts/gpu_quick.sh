#!/bin/bash
# quick check: parity subset + bench + optional ncu of kf (PROF="--workload W --m M")
mkdir -p gpurun_out
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ -n "$PROF" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kf_fused -s 2 -c 1 \
   -o gpurun_out/kf_prof python scripts/prof_driver.py $PROF > gpurun_out/ncu.log 2>&1
fi
