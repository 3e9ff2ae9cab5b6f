#!/bin/bash
# full GPU test suite + bench after the L2-read fix of PDL secondaries
mkdir -p gpurun_out/r02s2
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02s2
timeout 600 python -m pytest tests/test_gpu_repeat.py -q -p no:cacheprovider > $O/pytest_repeat.txt 2>&1; echo "rc=$?" >> $O/pytest_repeat.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > $O/pytest2.txt 2>&1
echo "pytest rc=$?" >> $O/pytest2.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench2.json 2> $O/bench2.err
echo "bench rc=$?" >> $O/bench2.err
