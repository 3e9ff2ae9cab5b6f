#!/bin/bash
mkdir -p gpurun_out/r02s2
O=gpurun_out/r02s2/dbg4.txt; : > $O
for L in "" build/var_KR_NOPDL/libms.so build/var_CG/libms.so; do
  for args in "fresh 16777216 256 1" "zero 16777216 256 0" "fresh 16777216 128 1"; do
    echo "== lib=$L $args" >> $O
    DBG_LIB=$L timeout 300 python scripts/dbg_r02s2c.py $args 2>&1 | grep -v Warn | cut -c1-200 >> $O
  done
done
for args in "fresh 33554432 32 1" "zero 33554432 32 0" "fresh 33554432 8 0"; do
  echo "== base $args" >> $O
  timeout 300 python scripts/dbg_r02s2c.py $args 2>&1 | grep -v Warn | cut -c1-200 >> $O
done
