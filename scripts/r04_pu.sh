#!/bin/bash
# push: lanes already in the new word need no atomic; unroll 1 / 4 (default) x straggler thresholds
mkdir -p gpurun_out
export MGK_MS_DIAG=1
for v in base pu1; do
  if [ $v = base ]; then unset MGK_LIB_PATH; else export MGK_LIB_PATH=build/var_$v/libmgk.so; fi
  for s in 8 16 32 64; do
    echo "== $v strag $s"; MGK_STRAG=$s timeout 600 python scripts/lanes_probe.py G4 10 2>&1 | grep "k=6\|rror" | cut -c1-900
  done
done
unset MGK_LIB_PATH
for s in 8 16 32 64; do echo "== G2 base strag $s"; MGK_STRAG=$s timeout 600 python scripts/lanes_probe.py G2 10 2>&1 | grep "k=6\|rror" | cut -c1-900; done
