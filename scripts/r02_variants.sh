#!/bin/bash
# A/B of compile-time LANES variants (build/var_*/libmgk.so, make variant ...)
mkdir -p gpurun_out
python scripts/lanes_probe.py both 16 > gpurun_out/var_base.log 2>&1
for v in build/var_*/libmgk.so; do
  n=$(basename $(dirname $v))
  MGK_LIB_PATH=$PWD/$v python scripts/lanes_probe.py both 16 > gpurun_out/$n.log 2>&1
done
grep -H "k=6" gpurun_out/var_*.log
