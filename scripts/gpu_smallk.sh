#!/bin/bash
# Tiny --steps / --warmup runs (the driver chooses K and W) at N = 1 and N = all GPUs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/sk_n1.log 2>&1; echo "rc=$?" >> gpurun_out/sk_n1.log
timeout 300 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/sk_n1b.log 2>&1; echo "rc=$?" >> gpurun_out/sk_n1b.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/sk_nN.log 2>&1; echo "rc=$?" >> gpurun_out/sk_nN.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus $N --impl reference --steps 5 --warmup 3 > gpurun_out/sk_ref.log 2>&1; echo "rc=$?" >> gpurun_out/sk_ref.log
