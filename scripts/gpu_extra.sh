#!/bin/bash
# f1 refresh (ResNet-50 iterations at N = 1, 2, 4), an odd-k bench line (N = 3), smoke.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
python paper_1711_04325_b200/build.py > gpurun_out/final/build_e.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final/smoke.log
CUDA_VISIBLE_DEVICES=0,1,2 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 3 --master-addr 127.0.0.1 --master-port 29573 bench.py --gpus 3 > gpurun_out/final/n3.log 2>&1; echo "rc=$?" >> gpurun_out/final/n3.log
timeout 600 python tools/resnet_iteration.py > gpurun_out/final/resnet_n1.log 2>&1; echo "rc=$?" >> gpurun_out/final/resnet_n1.log
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n tools/resnet_iteration.py > gpurun_out/final/resnet_n$n.log 2>&1; echo "rc=$?" >> gpurun_out/final/resnet_n$n.log
done
