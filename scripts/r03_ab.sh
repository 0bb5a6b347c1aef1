#!/bin/bash
# A/B: degree-ordered ids (MGK_RELABEL=1 in-degree / 2 out-degree) x LANES hub words in shared memory
mkdir -p gpurun_out
export MGK_MS_DIAG=1
timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/ab_base.log 2>&1
MGK_RELABEL=2 MGK_PROBE_HUB=1 timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/ab_r2_nohub.log 2>&1
MGK_RELABEL=2 timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/ab_r2_hub.log 2>&1
MGK_RELABEL=1 timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/ab_r1_hub.log 2>&1
MGK_RELABEL=2 timeout 900 python -m pytest -q -m gpu tests/test_gpu_parity.py -x > gpurun_out/ab_r2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_r2_tests.log
for f in gpurun_out/ab_*.log; do echo "== $f"; grep -h "k2 300\|k=6\|rc=\|passed\|failed\|Error" $f | cut -c1-400; done
