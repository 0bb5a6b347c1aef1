#!/bin/bash
# A/B: dense/packed pulls by unsettled count + streamed frontier clears, vs HEAD; minb4 variant; parity
mkdir -p gpurun_out
export MGK_MS_DIAG=1
for rep in 1 2; do
timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/pk2_base$rep.log 2>&1
MGK_LIB_PATH=$PWD/build/var_head/libmgk.so timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/pk2_head$rep.log 2>&1
MGK_LIB_PATH=$PWD/build/var_minb4/libmgk.so timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/pk2_minb4$rep.log 2>&1
done
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_configs.py tests/test_gpu_parity.py -x > gpurun_out/pk2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pk2_tests.log
for f in gpurun_out/pk2_*.log; do echo "== $f"; grep -h "k=6\|Error\|rror" $f | cut -c1-420; done
tail -3 gpurun_out/pk2_tests.log
