#!/bin/bash
# A/B of the split first pull (hub_deg thresholds; 0 = whole pulls) + LANES parity
mkdir -p gpurun_out
export MGK_MS_DIAG=1
for d in 0 64 32 128 256; do
  MGK_HUB_DEG=$d timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/split_d$d.log 2>&1
done
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_configs.py tests/test_gpu_parity.py -x > gpurun_out/split_tests.log 2>&1; echo "rc=$?" >> gpurun_out/split_tests.log
for f in gpurun_out/split_d*.log; do echo "== $f"; grep -h "k2 300\|k=6\|Error\|rror" $f | cut -c1-420; done
tail -3 gpurun_out/split_tests.log
