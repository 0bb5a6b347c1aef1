#!/bin/bash
# SWAR lane counting: sections probe + LANES / config parity
mkdir -p gpurun_out
MGK_MS_DIAG=1 python scripts/sched_probe.py G4 > gpurun_out/cnt_sched.log 2>&1
MGK_MS_DIAG=1 python scripts/sched_probe.py G2 >> gpurun_out/cnt_sched.log 2>&1
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_configs.py tests/test_gpu_parity.py -x > gpurun_out/cnt_tests.log 2>&1; echo "rc=$?" >> gpurun_out/cnt_tests.log
grep " ms " gpurun_out/cnt_sched.log | cut -c1-250; tail -3 gpurun_out/cnt_tests.log
