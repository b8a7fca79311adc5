#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_n1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n1.log
timeout 300 python bench.py --no-cpu-baseline --t-start 1000 > gpurun_out/bench_n1_sgd.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n1_sgd.log
timeout 300 python bench.py --mode fused --no-cpu-baseline > gpurun_out/bench_n1_fused.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n1_fused.log
