#!/bin/bash
# full GPU test suite, smoke, default bench line with sweep, launch list of the default bench
mkdir -p gpurun_out/r02s3f
export PATH=/usr/local/cuda/bin:$PATH
O=gpurun_out/r02s3f
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/full_smoke.txt 2>&1; echo "smoke rc=$?" >> $O/full_smoke.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > $O/full_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/full_pytest.txt
timeout 1200 python bench.py --steps 50 --warmup 5 > $O/full_bench.json 2> $O/full_bench.err; echo "bench rc=$?" >> $O/full_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  python bench.py --steps 5 --warmup 3 --no-sweep --no-cpu-baseline > $O/full_launches.csv 2> $O/full_launches.err
