#!/bin/bash
# push-unroll variants with straggler lanes (A/B), the reference arm, then ncu captures of the dominant kernels on the
# current code (one GPU, one process at a time) + the bench's launch list
mkdir -p gpurun_out
export MGK_MS_DIAG=1
for v in base pu2 pu4; do
  if [ $v = base ]; then unset MGK_LIB_PATH; else export MGK_LIB_PATH=build/var_$v/libmgk.so; fi
  echo "== $v"; timeout 600 python scripts/lanes_probe.py G4 10 2>&1 | grep "bits=\|rror" | cut -c1-900
done
unset MGK_LIB_PATH MGK_MS_DIAG
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
head -c 300 gpurun_out/bench_ref.json; echo
export MGK_NONCOOP=1   # ncu does not intercept cooperative launches
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:ms_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/r04b_ms_cfg4_k6 -f python scripts/prof_target.py G4 6 10 > gpurun_out/ncu_ms_cfg4.log 2>&1
timeout 600 $NCU -k regex:ms_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/r04b_ms_cfg3_k6 -f python scripts/prof_target.py G2 6 10 > gpurun_out/ncu_ms_cfg3.log 2>&1
timeout 900 $NCU -k regex:k2_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/r04b_k2_cfg4_k2 -f python scripts/prof_target.py G4 2 300 > gpurun_out/ncu_k2_cfg4.log 2>&1
timeout 600 $NCU -k regex:k2_kernel --launch-skip 2 --launch-count 1 -o gpurun_out/r04b_k2_cfg2_k2 -f python scripts/prof_target.py G2 2 300 > gpurun_out/ncu_k2_cfg2.log 2>&1
timeout 900 $NCU -k regex:ms_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/r04b_ms_cfg5_k3 -f python scripts/prof_target.py G2 3 65536 8 2 > gpurun_out/ncu_ms_cfg5.log 2>&1
unset MGK_NONCOOP
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r04b_launches_cfg4.csv \
    python bench.py --steps 2 --warmup 3 --no-extras --no-cpu > gpurun_out/ncu_launches.log 2>&1
ls -la gpurun_out | grep r04b
