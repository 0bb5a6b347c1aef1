#!/bin/bash
mkdir -p gpurun_out
export MGK_NONCOOP=1
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:ms_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/ms_cfg4_k6 -f python scripts/prof_target.py G4 6 10 > gpurun_out/ncu_ms_cfg4.log 2>&1
$NCU -k regex:ms_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/ms_cfg3_k6 -f python scripts/prof_target.py G2 6 10 > gpurun_out/ncu_ms_cfg3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_cfg4.csv \
    python bench.py --steps 2 --warmup 3 --no-extras --no-cpu > gpurun_out/ncu_launches.log 2>&1
ls gpurun_out
