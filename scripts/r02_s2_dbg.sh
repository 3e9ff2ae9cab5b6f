#!/bin/bash
mkdir -p gpurun_out/r02s2
export PATH=/usr/local/cuda/bin:$PATH
timeout 2400 python scripts/dbg_r02s2.py > gpurun_out/r02s2/dbg.txt 2>&1
