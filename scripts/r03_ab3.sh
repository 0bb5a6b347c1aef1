#!/bin/bash
# A/B: buffered candidate packing + dense finalize + streamed frontier clears, vs HEAD; parity
mkdir -p gpurun_out
export MGK_MS_DIAG=1
for rep in 1 2; do
timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/ab3_base$rep.log 2>&1
MGK_LIB_PATH=$PWD/build/var_head/libmgk.so timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/ab3_head$rep.log 2>&1
done
MGK_HUB_DEG=256 timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/ab3_split256.log 2>&1
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_configs.py tests/test_gpu_parity.py -x > gpurun_out/ab3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab3_tests.log
for f in gpurun_out/ab3_*.log; do echo "== $f"; grep -h "k=6\|Error\|rror" $f | cut -c1-420; done
tail -3 gpurun_out/ab3_tests.log
