#!/bin/bash
# Config C5 (whole 90-epoch schedule, ResNet-152 buffer, BN sync per epoch) at N = all GPUs, and at N = 1.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $N --depth 152 --full-schedule --no-profile > gpurun_out/c5_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/c5_n$N.log
timeout 600 python bench.py --depth 152 --full-schedule --no-profile --no-cpu-baseline > gpurun_out/c5_n1.log 2>&1; echo "rc=$?" >> gpurun_out/c5_n1.log
