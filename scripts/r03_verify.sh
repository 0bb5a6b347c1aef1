#!/bin/bash
# probe (10-bit and 16-bit words) + the LANES / config GPU tests
mkdir -p gpurun_out
MGK_MS_DIAG=1 timeout 900 python scripts/lanes_probe.py both 10 16 > gpurun_out/verify_probe.log 2>&1
timeout 1500 python -m pytest -q -m gpu tests/test_gpu_configs.py tests/test_gpu_parity.py -x > gpurun_out/verify_tests.log 2>&1; echo "rc=$?" >> gpurun_out/verify_tests.log
grep -h "k=6\|k=3\|Error\|rror" gpurun_out/verify_probe.log | cut -c1-300
tail -3 gpurun_out/verify_tests.log
