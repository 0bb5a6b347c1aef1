#!/bin/bash
# state check after a container restore: tests + smoke + bench + LANES per-hop probe
mkdir -p gpurun_out
SKIP_REF=1 bash scripts/r02_check.sh
MGK_MS_DIAG=1 timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/lanes_diag.log 2>&1
tail -3 gpurun_out/gputests.log; cat gpurun_out/smoke.log | tail -2; tail -2 gpurun_out/bench.err; grep k= gpurun_out/lanes_diag.log
