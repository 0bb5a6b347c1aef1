#!/bin/bash
# A/B: rematerialised L2 policies (48 regs) and 6 CTAs/SM (40 regs) vs HEAD
mkdir -p gpurun_out
export MGK_MS_DIAG=1
for rep in 1 2; do
timeout 600 python scripts/lanes_probe.py both 10 > gpurun_out/ab7_base$rep.log 2>&1
MGK_LIB_PATH=$PWD/build/var_minb6/libmgk.so timeout 600 python scripts/lanes_probe.py both 10 > gpurun_out/ab7_minb6$rep.log 2>&1
MGK_LIB_PATH=$PWD/build/var_head/libmgk.so timeout 600 python scripts/lanes_probe.py both 10 > gpurun_out/ab7_head$rep.log 2>&1
done
for f in gpurun_out/ab7_*.log; do echo "== $f"; grep -h "k=6\|Error\|rror" $f | cut -c1-420; done
