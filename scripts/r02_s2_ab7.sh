#!/bin/bash
mkdir -p gpurun_out/r02s2
O=gpurun_out/r02s2
timeout 900 python -m pytest tests/test_gpu_splitters.py -q -p no:cacheprovider -x > $O/ab7_pytest.txt 2>&1; echo "rc=$?" >> $O/ab7_pytest.txt
timeout 1200 python scripts/ab.py 'ms_keys_large:1024,ms_keys_large:4096,ms_keys_large:65536,ms_pairs_large:4096' > $O/ab7.txt 2>&1
