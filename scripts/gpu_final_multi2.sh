#!/bin/bash
# Final multi-GPU bench lines on a 4-GPU box: N = 2 (GPUs 0,1) and N = 4, ResNet-50 and
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
python paper_1711_04325_b200/build.py > gpurun_out/final/build_m.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 400 $TR --nproc-per-node 2 --master-port 29571 bench.py --gpus 2 > gpurun_out/final/n2.log 2>&1; echo "rc=$?" >> gpurun_out/final/n2.log
timeout 400 $TR --nproc-per-node 4 --master-port 29572 bench.py --gpus 4 > gpurun_out/final/n4.log 2>&1; echo "rc=$?" >> gpurun_out/final/n4.log
timeout 400 $TR --nproc-per-node 4 --master-port 29573 bench.py --gpus 4 --depth 152 > gpurun_out/final/n4_r152.log 2>&1; echo "rc=$?" >> gpurun_out/final/n4_r152.log
echo done > gpurun_out/final/done_m.txt
