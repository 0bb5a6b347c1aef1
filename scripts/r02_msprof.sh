#!/bin/bash
mkdir -p gpurun_out
MGK_MS_DIAG=1 python scripts/lanes_probe.py both 16 > gpurun_out/lanes_diag.log 2>&1
export MGK_NONCOOP=1
ncu --set full --clock-control none --import-source on -k regex:ms_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/ms_cfg4_k6 -f python scripts/prof_target.py G4 6 10 > gpurun_out/ncu_ms_cfg4.log 2>&1
tail -2 gpurun_out/ncu_ms_cfg4.log
