#!/bin/bash
mkdir -p gpurun_out/r02s2
timeout 900 python scripts/dbg_r02s2b.py > gpurun_out/r02s2/dbg2.txt 2>&1
timeout 1500 python scripts/dbg_sweep.py > gpurun_out/r02s2/dbg_sweep.txt 2>&1
