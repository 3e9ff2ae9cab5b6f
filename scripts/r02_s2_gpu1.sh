#!/bin/bash
# round 2 session 2, call 1: state of HEAD (GPU tests, smoke, bench line)
mkdir -p gpurun_out/r02s2
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02s2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x --timeout 900 > $O/pytest.txt 2>&1
echo "pytest rc=$?" >> $O/pytest.txt
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/bench.err
