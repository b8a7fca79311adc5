#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
UBENCH_ITERS=2000 timeout 300 ./tools/ubench > gpurun_out/ubench_2k.log 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,clocks_event_reasons.active --format=csv -lms 100 > gpurun_out/ub_clocks.csv &
SMI=$!
UBENCH_ITERS=2000 timeout 300 ./tools/ubench > gpurun_out/ubench_2k_b.log 2>&1
kill $SMI
timeout 300 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/bench_200.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 5000 > gpurun_out/bench_5000.log 2>&1
