#!/bin/bash
# full round-end style check: GPU tests, smoke, bench (our arm), bench (reference arm)
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests > gpurun_out/gputests.log 2>&1; echo "gputests rc=$?" >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
tail -3 gpurun_out/gputests.log; tail -1 gpurun_out/smoke.log
python scripts/bench_summary.py gpurun_out/bench.json 2>/dev/null | head -30 || head -c 1500 gpurun_out/bench.json
head -c 600 gpurun_out/bench_ref.json
