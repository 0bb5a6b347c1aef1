#!/bin/bash
# top4 (dense array of every vertex's first four in-neighbours) A/B, parity tests, bench
mkdir -p gpurun_out
export MGK_MS_DIAG=1
echo "== top4"; timeout 600 python scripts/lanes_probe.py both 10 2>&1 | grep "bits=\|rror" | cut -c1-900
echo "== no top4"; MGK_NO_TOP4=1 timeout 600 python scripts/lanes_probe.py both 10 2>&1 | grep "bits=\|rror" | cut -c1-900
unset MGK_MS_DIAG
timeout 1500 python -m pytest -q -m gpu tests/test_gpu_configs.py tests/test_gpu_parity.py -x > gpurun_out/top4_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/top4_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/bench.json
