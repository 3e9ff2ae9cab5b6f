#!/bin/bash
mkdir -p gpurun_out/r02s2
timeout 1200 python scripts/ab.py 'ms_keys:32,ms_keys:24,ms_pairs:32,ms_keys:32' 'exp=0;exp=1;exp=0;exp=1' > gpurun_out/r02s2/ab8.txt 2>&1
