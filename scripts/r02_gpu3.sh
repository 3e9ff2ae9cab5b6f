#!/bin/bash
mkdir -p gpurun_out/r02
export PATH=/usr/local/cuda/bin:$PATH
TAG=${TAG:-gpu3}
python scripts/dbg_wide.py > gpurun_out/r02/${TAG}_dbg.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rank_modes.py -x -q -p no:cacheprovider > gpurun_out/r02/${TAG}_pytest.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/${TAG}_pytest.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02/${TAG}_bench.json 2> gpurun_out/r02/${TAG}_bench.err
SPECS="kf_meta_wide:ms_keys:256:${TAG}_kfw_keys256 kf_meta_wide:ms_pairs_c3:256:${TAG}_kfw_pairs256 km_meta_wide:ms_keys:256:${TAG}_kmw_keys256" bash scripts/r02_prof.sh
