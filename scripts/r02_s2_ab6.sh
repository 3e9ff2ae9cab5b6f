#!/bin/bash
mkdir -p gpurun_out/r02s2
O=gpurun_out/r02s2
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x --timeout 900 > $O/ab6_pytest.txt 2>&1; echo "rc=$?" >> $O/ab6_pytest.txt
timeout 1200 python scripts/ab.py 'ms_keys:2,ms_keys:4,ms_keys:8,ms_keys:16,ms_keys:32,ms_pairs:2,ms_pairs:16,ms_pairs:32,ms_keys:64,ms_keys:256,ms_pairs:256,ms_pairs_c3:256,sort_keys:256,sort_pairs:256' > $O/ab6.txt 2>&1
python -c "
import torch, bench, json
print(json.dumps(bench.c1_latency(torch.device('cuda', 0))))" >> $O/ab6.txt 2>&1
