#!/bin/bash
# straggler lanes (MGK_STRAG): lanes_probe per-hop split at several thresholds vs the build before it, then parity tests with it on
mkdir -p gpurun_out
export MGK_MS_DIAG=1
echo "== base (HEAD build)"; MGK_LIB_PATH=build/var_base/libmgk.so timeout 600 python scripts/lanes_probe.py both 10 2>&1 | grep "bits=\|rror" | cut -c1-900
for s in 0 16 64 256 1024; do
  echo "== strag $s"; MGK_STRAG=$s timeout 600 python scripts/lanes_probe.py both 10 2>&1 | grep "bits=\|rror" | cut -c1-900
done
unset MGK_MS_DIAG
MGK_STRAG=64 timeout 1500 python -m pytest -q -m gpu tests/test_gpu_configs.py tests/test_gpu_parity.py -x > gpurun_out/strag_tests.log 2>&1; echo "tests(strag 64) rc=$?"
tail -3 gpurun_out/strag_tests.log
