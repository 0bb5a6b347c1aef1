#!/bin/bash
# A/B: flattened per-word pull scans (default) vs a lane per vertex (var_noflat), prefix 8/16/32; split pull on/off
mkdir -p gpurun_out
export MGK_MS_DIAG=1
timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/flat_base.log 2>&1
for v in noflat pre16 pre32; do
  MGK_LIB_PATH=$PWD/build/var_$v/libmgk.so timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/flat_$v.log 2>&1
done
MGK_HUB_DEG=256 timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/flat_split256.log 2>&1
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_configs.py tests/test_gpu_parity.py -x > gpurun_out/flat_tests.log 2>&1; echo "rc=$?" >> gpurun_out/flat_tests.log
for f in gpurun_out/flat_*.log; do echo "== $f"; grep -h "k=6\|Error\|rror" $f | cut -c1-420; done
tail -3 gpurun_out/flat_tests.log
