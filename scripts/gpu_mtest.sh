#!/bin/bash
# Multi-GPU parity test + traced bench at N = all visible GPUs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_multigpu.py -q > gpurun_out/pytest_mgpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mgpu.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29507 bench.py --gpus $N --trace --steps 1000 > gpurun_out/bench_trace_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/bench_trace_n$N.log
