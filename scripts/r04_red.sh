#!/bin/bash
# mixed hop's push with fire-and-forget ORs and no list: thresholds, parity tests, bench
mkdir -p gpurun_out
export MGK_MS_DIAG=1
for s in 16 32 64; do echo "== G4 strag $s"; MGK_STRAG=$s timeout 600 python scripts/lanes_probe.py G4 10 2>&1 | grep "bits=\|rror" | cut -c1-900; done
for s in 16 32 64; do echo "== G2 strag $s"; MGK_STRAG=$s timeout 600 python scripts/lanes_probe.py G2 10 2>&1 | grep "bits=\|rror" | cut -c1-900; done
unset MGK_MS_DIAG
for s in 32 64; do
MGK_STRAG=$s timeout 1500 python -m pytest -q -m gpu tests/test_gpu_configs.py tests/test_gpu_parity.py -x > gpurun_out/red_tests_$s.log 2>&1; echo "tests strag $s rc=$?"
tail -3 gpurun_out/red_tests_$s.log
done
