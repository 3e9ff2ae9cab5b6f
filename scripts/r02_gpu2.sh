#!/bin/bash
# round 2: parity of the wide (m > 32) pipeline + bench sweep
mkdir -p gpurun_out/r02
export PATH=/usr/local/cuda/bin:$PATH
TAG=${TAG:-gpu2}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rank_modes.py -x -q -p no:cacheprovider > gpurun_out/r02/${TAG}_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/${TAG}_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02/${TAG}_bench.json 2> gpurun_out/r02/${TAG}_bench.err
