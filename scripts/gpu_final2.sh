#!/bin/bash
# Headline lines: N = 1 default (with CPU baseline), N = 2 (all GPUs of a 2-GPU box).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 600 python bench.py > gpurun_out/final_n1.log 2>&1; echo "rc=$?" >> gpurun_out/final_n1.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $N > gpurun_out/final_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/final_n$N.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/final_ref_n1.log 2>&1; echo "rc=$?" >> gpurun_out/final_ref_n1.log
