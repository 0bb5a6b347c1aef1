#!/bin/bash
# A/B: 10-bit lane words (three per 32-bit word) vs 16-bit for the 10-seed batches; full GPU tests
mkdir -p gpurun_out
export MGK_MS_DIAG=1
timeout 900 python scripts/lanes_probe.py both 10 16 10 > gpurun_out/b10_probe.log 2>&1
unset MGK_MS_DIAG
timeout 1500 python -m pytest -q -m gpu tests -x > gpurun_out/b10_tests.log 2>&1; echo "rc=$?" >> gpurun_out/b10_tests.log
grep -h "k=6\|k=3\|Error\|rror" gpurun_out/b10_probe.log | cut -c1-420
tail -3 gpurun_out/b10_tests.log
