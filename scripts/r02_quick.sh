#!/bin/bash
# quick A/B: LANES probe + the LANES / config parity tests
mkdir -p gpurun_out
python scripts/lanes_probe.py both ${BITS:-16} > gpurun_out/lanes_probe.log 2>&1
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_configs.py tests/test_gpu_parity.py ${PYTEST_EXTRA:-} > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
tail -2 gpurun_out/quick_tests.log
