#!/bin/bash
# Round-2 first check on the box: host facts, GPU tests, smoke, a short bench.
mkdir -p gpurun_out
bash scripts/box_probe.sh > gpurun_out/box_probe.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "gputests rc=$?" >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/gputests.log
