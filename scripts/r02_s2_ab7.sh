#!/bin/bash
mkdir -p gpurun_out/r02s2
O=gpurun_out/r02s2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_skew.py tests/test_gpu_repeat.py tests/test_gpu_splitters.py tests/test_gpu_sharded.py -q -p no:cacheprovider -x > $O/ab7_pytest.txt 2>&1; echo "rc=$?" >> $O/ab7_pytest.txt
timeout 1200 python scripts/ab.py 'ms_keys_spl:32,ms_keys_spl:256,ms_pairs_spl:256,ms_keys:8,ms_keys:32,ms_keys:256,ms_pairs_c3:256' > $O/ab7.txt 2>&1
