#!/bin/bash
# A/B of compile-time LANES variants (build/var_*/libmgk.so) against the default build
mkdir -p gpurun_out
export MGK_MS_DIAG=1
timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/var_base.log 2>&1
for n in step8 wpr4 step8wpr4 pre16 blk384; do
  MGK_LIB_PATH=$PWD/build/var_$n/libmgk.so timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/var_$n.log 2>&1
done
timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/var_base2.log 2>&1
for f in gpurun_out/var_*.log; do echo "== $f"; grep -h "k=6\|Error\|rror" $f | cut -c1-300; done
