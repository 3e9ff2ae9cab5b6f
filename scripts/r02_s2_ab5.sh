#!/bin/bash
mkdir -p gpurun_out/r02s2
timeout 1200 python scripts/ab.py 'ms_pairs_c3:256,ms_pairs:256,ms_keys:256,ms_pairs:128' 'exp=0;exp=1;exp=2;exp=3' > gpurun_out/r02s2/ab5.txt 2>&1
