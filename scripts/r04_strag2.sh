#!/bin/bash
# straggler lanes on by default: CTAs per SM (5 / 6) and thresholds, then all GPU tests and the bench
mkdir -p gpurun_out
export MGK_MS_DIAG=1
for mb in 6 5; do for s in 32 64 128; do
  echo "== mb $mb strag $s"; MGK_MS_MB=$mb MGK_STRAG=$s timeout 600 python scripts/lanes_probe.py G4 10 2>&1 | grep "bits=\|rror" | cut -c1-900
done; done
echo "== G2 mb 5 (default) / 6, strag 64"
MGK_STRAG=64 timeout 600 python scripts/lanes_probe.py G2 10 2>&1 | grep "bits=\|rror" | cut -c1-900
MGK_MS_MB=6 MGK_STRAG=64 timeout 600 python scripts/lanes_probe.py G2 10 2>&1 | grep "bits=\|rror" | cut -c1-900
unset MGK_MS_DIAG
timeout 1500 python -m pytest -q -m gpu tests > gpurun_out/gputests.log 2>&1; echo "gputests rc=$?" >> gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/bench.json
