#!/bin/bash
# A/B of the LANES kernel's loop-carried state (spills of the 6-CTA instance): current build vs the r04a and
# 0b27941 builds of mgk_ms.cu (build/var_r04a, build/var_head), then the LANES parity tests and the bench
mkdir -p gpurun_out
export MGK_MS_DIAG=1
for v in base r04a head; do
  if [ $v = base ]; then unset MGK_LIB_PATH; else export MGK_LIB_PATH=build/var_$v/libmgk.so; fi
  echo "== $v"; timeout 600 python scripts/lanes_probe.py both 10 2>&1 | grep "bits=\|k2 300" | cut -c1-900
done
unset MGK_LIB_PATH MGK_MS_DIAG
timeout 1500 python -m pytest -q -m gpu tests/test_gpu_configs.py tests/test_gpu_parity.py -x > gpurun_out/spill_tests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/spill_tests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/bench.json
