#!/bin/bash
# End-of-round check on a 4-GPU box: full GPU suite, smoke, N = 2 and N = 4 bench lines.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
python paper_1711_04325_b200/build.py > gpurun_out/final/build_c.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final/smoke.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
CUDA_VISIBLE_DEVICES=0,1 timeout 400 $TR --nproc-per-node 2 --master-port 29571 bench.py --gpus 2 > gpurun_out/final/n2.log 2>&1; echo "rc=$?" >> gpurun_out/final/n2.log
timeout 400 $TR --nproc-per-node 4 --master-port 29572 bench.py --gpus 4 > gpurun_out/final/n4.log 2>&1; echo "rc=$?" >> gpurun_out/final/n4.log
