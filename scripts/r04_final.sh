#!/bin/bash
# final state: GPU tests, smoke, bench (both arms), ncu of the LANES kernel (cfg4, cfg3) and the launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -m gpu tests > gpurun_out/gputests.log 2>&1; echo "gputests rc=$?" >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
tail -3 gpurun_out/gputests.log; tail -2 gpurun_out/smoke.log
python scripts/bench_summary.py gpurun_out/bench.json
head -c 400 gpurun_out/bench_ref.json; echo
export MGK_NONCOOP=1
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:ms_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/r04e_ms_cfg4_k6 -f python scripts/prof_target.py G4 6 10 > gpurun_out/ncu_ms_cfg4.log 2>&1
timeout 600 $NCU -k regex:ms_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/r04e_ms_cfg3_k6 -f python scripts/prof_target.py G2 6 10 > gpurun_out/ncu_ms_cfg3.log 2>&1
unset MGK_NONCOOP
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r04e_launches_cfg4.csv \
    python bench.py --steps 2 --warmup 3 --no-extras --no-cpu > gpurun_out/ncu_launches.log 2>&1
ls -la gpurun_out | grep r04e
