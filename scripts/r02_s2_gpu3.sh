#!/bin/bash
mkdir -p gpurun_out/r02s2
O=gpurun_out/r02s2
timeout 1500 python -m pytest tests/test_gpu_splitters.py -q -p no:cacheprovider -x > $O/gpu3_split.txt 2>&1; echo "rc=$?" >> $O/gpu3_split.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 --deselect tests/test_gpu_splitters.py > $O/gpu3_all.txt 2>&1; echo "rc=$?" >> $O/gpu3_all.txt
