#!/bin/bash
# A/B: L1 eviction priorities (gathers evict_last; in-list reads evict_first), with and without out-degree relabelling
mkdir -p gpurun_out
export MGK_MS_DIAG=1
run() { timeout 600 python scripts/lanes_probe.py both 10 > gpurun_out/ab8_$1.log 2>&1; }
run base
MGK_LIB_PATH=$PWD/build/var_l1g/libmgk.so run l1g
MGK_LIB_PATH=$PWD/build/var_l1gri/libmgk.so run l1gri
MGK_RELABEL=2 run r2
MGK_RELABEL=2 MGK_LIB_PATH=$PWD/build/var_l1g/libmgk.so run r2_l1g
MGK_RELABEL=2 MGK_LIB_PATH=$PWD/build/var_l1gri/libmgk.so run r2_l1gri
for f in gpurun_out/ab8_*.log; do echo "== $f"; grep -h "k=6\|Error\|rror" $f | cut -c1-300; done
