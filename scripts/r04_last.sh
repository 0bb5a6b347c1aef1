#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python scripts/bench_summary.py gpurun_out/bench.json
timeout 1500 python -m pytest -q -m gpu tests > gpurun_out/gputests.log 2>&1; echo "gputests rc=$?" >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -3 gpurun_out/gputests.log; tail -2 gpurun_out/smoke.log
