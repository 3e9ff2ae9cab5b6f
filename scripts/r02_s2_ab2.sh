#!/bin/bash
mkdir -p gpurun_out/r02s2
timeout 900 python -m pytest tests/test_gpu_repeat.py tests/test_gpu_rank_modes.py tests/test_gpu_parity.py -q -p no:cacheprovider -x > gpurun_out/r02s2/ab2_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02s2/ab2_pytest.txt
timeout 1200 python scripts/ab.py 'ms_keys:4,ms_keys:8,ms_keys:16,ms_keys:32,ms_pairs:32,ms_keys:64,ms_keys:128,ms_keys:256,ms_pairs:64,ms_pairs:256,ms_pairs_c3:256,sort_keys:256,sort_pairs:256' > gpurun_out/r02s2/ab2.txt 2>&1
