#!/bin/bash
# A/B: software-pipelined pull rounds (var_pipe), 6 CTAs/SM (var_minb6) vs default; 10-bit words
mkdir -p gpurun_out
export MGK_MS_DIAG=1
for rep in 1 2; do
timeout 600 python scripts/lanes_probe.py both 10 > gpurun_out/ab5_base$rep.log 2>&1
for n in pipe minb6; do
  MGK_LIB_PATH=$PWD/build/var_$n/libmgk.so timeout 600 python scripts/lanes_probe.py both 10 > gpurun_out/ab5_$n$rep.log 2>&1
done
done
for f in gpurun_out/ab5_*.log; do echo "== $f"; grep -h "k=6\|Error\|rror" $f | cut -c1-420; done
