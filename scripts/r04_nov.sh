#!/bin/bash
# mixed hop's push without the visited-word gather (finalize masks): probe, parity tests
mkdir -p gpurun_out
export MGK_MS_DIAG=1
for s in 16 32; do echo "== G4 strag $s"; MGK_STRAG=$s timeout 600 python scripts/lanes_probe.py both 10 2>&1 | grep "k=6\|rror" | cut -c1-900; done
unset MGK_MS_DIAG
timeout 1500 python -m pytest -q -m gpu tests/test_gpu_configs.py tests/test_gpu_parity.py -x > gpurun_out/nov_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/nov_tests.log
