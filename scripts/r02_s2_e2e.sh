#!/bin/bash
mkdir -p gpurun_out/r02s2
O=gpurun_out/r02s2
: > $O/e2e.txt
for w in ms_keys ms_pairs sort_keys ms_pairs_c3; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-sweep --no-cpu-baseline >> $O/e2e.txt 2>> $O/e2e.err
done
python -c "
import torch, bench, json
print(json.dumps(bench.c1_latency(torch.device('cuda', 0))))" >> $O/e2e.txt 2>&1
