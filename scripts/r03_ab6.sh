#!/bin/bash
# A/B: short-list / long-list candidate rounds vs HEAD (one buffer); LANES parity
mkdir -p gpurun_out
export MGK_MS_DIAG=1
for rep in 1 2; do
timeout 600 python scripts/lanes_probe.py both 10 > gpurun_out/ab6_base$rep.log 2>&1
MGK_LIB_PATH=$PWD/build/var_head/libmgk.so timeout 600 python scripts/lanes_probe.py both 10 > gpurun_out/ab6_head$rep.log 2>&1
done
unset MGK_MS_DIAG
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_configs.py tests/test_gpu_parity.py -x > gpurun_out/ab6_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab6_tests.log
for f in gpurun_out/ab6_*.log; do echo "== $f"; grep -h "k=6\|Error\|rror" $f | cut -c1-420; done
tail -3 gpurun_out/ab6_tests.log
