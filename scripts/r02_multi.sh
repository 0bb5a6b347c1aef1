#!/bin/bash
# functional check of the N>1 bench path on a one-GPU box (gloo, ranks share the GPU)
mkdir -p gpurun_out
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_parity.py -k "replicas or multi" > gpurun_out/multi_tests.log 2>&1; echo "rc=$?" >> gpurun_out/multi_tests.log
MGK_BENCH_DRYRUN=1 timeout 1200 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_dry2.json 2> gpurun_out/bench_dry2.err; echo "rc=$?" >> gpurun_out/bench_dry2.err
tail -2 gpurun_out/multi_tests.log; tail -3 gpurun_out/bench_dry2.err
