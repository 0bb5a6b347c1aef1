#!/bin/bash
# global out-degree / in-degree relabelling on the current LANES code (A/B), then ncu of ms_kernel (G4 k=6, 10 seeds)
mkdir -p gpurun_out
export MGK_MS_DIAG=1
MGK_RELABEL=2 timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/p_r2.log 2>&1
MGK_RELABEL=1 timeout 600 python scripts/lanes_probe.py both 16 > gpurun_out/p_r1.log 2>&1
unset MGK_MS_DIAG
export MGK_NONCOOP=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ms_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/r03_ms_cfg4_k6 -f python scripts/prof_target.py G4 6 10 > gpurun_out/ncu_ms_cfg4.log 2>&1
for f in gpurun_out/p_*.log; do echo "== $f"; grep -h "k2 300\|k=6\|Error\|rror" $f | cut -c1-420; done
tail -2 gpurun_out/ncu_ms_cfg4.log
