#!/bin/bash
mkdir -p gpurun_out
for v in base k2b384 k2b256; do
  if [ $v = base ]; then unset MGK_LIB_PATH; else export MGK_LIB_PATH=build/var_$v/libmgk.so; fi
  echo "== $v"; timeout 600 python scripts/k2ab.py G2 G4 2>&1 | tail -3
done
echo "== lanes diag"; MGK_MS_DIAG=1 timeout 600 python scripts/lanes_probe.py G4 10 2>&1 | tail -4 | cut -c1-900
