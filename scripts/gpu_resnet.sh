#!/bin/bash
# f1: ResNet-50 synthetic iterations at N = 1, 2, 4 (all GPUs of the box).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 600 python tools/resnet_iteration.py > gpurun_out/resnet_n1.log 2>&1; echo "rc=$?" >> gpurun_out/resnet_n1.log
for n in 2 4; do
  if [ "$N" -ge "$n" ]; then
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n tools/resnet_iteration.py > gpurun_out/resnet_n$n.log 2>&1; echo "rc=$?" >> gpurun_out/resnet_n$n.log
  fi
done
