#!/bin/bash
# A/B: split / per-lane modes removed (fewer spills) vs the previous commit; 64-register variant; parity
mkdir -p gpurun_out
export MGK_MS_DIAG=1
for rep in 1 2; do
timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/ab4_base$rep.log 2>&1
MGK_LIB_PATH=$PWD/build/var_prev/libmgk.so timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/ab4_prev$rep.log 2>&1
MGK_LIB_PATH=$PWD/build/var_minb4/libmgk.so timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/ab4_minb4$rep.log 2>&1
done
timeout 1500 python -m pytest -q -m gpu tests -x > gpurun_out/ab4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab4_tests.log
for f in gpurun_out/ab4_*.log; do echo "== $f"; grep -h "k=6\|Error\|rror" $f | cut -c1-420; done
tail -3 gpurun_out/ab4_tests.log
