#!/bin/bash
# dense-few finalize threshold A/B (n/32 default vs n/8, n/16); LANES parity tests
mkdir -p gpurun_out
export MGK_MS_DIAG=1
for v in base dd8 dd16; do
  if [ $v = base ]; then unset MGK_LIB_PATH; else export MGK_LIB_PATH=build/var_$v/libmgk.so; fi
  echo "== $v"; timeout 600 python scripts/lanes_probe.py both 10 2>&1 | grep "bits=" | cut -c1-700
done
unset MGK_LIB_PATH MGK_MS_DIAG
timeout 1500 python -m pytest -q -m gpu tests/test_gpu_configs.py tests/test_gpu_parity.py -x > gpurun_out/push_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/push_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/bench.json
