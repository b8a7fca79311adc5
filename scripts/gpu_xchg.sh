#!/bin/bash
# lmsgd_exchange: parity (k=1 and all GPUs) and the bench line at N = all GPUs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
python paper_1711_04325_b200/build.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "exchange" > gpurun_out/px.log 2>&1; echo "rc=$?" >> gpurun_out/px.log
timeout 900 python -m pytest tests/test_multigpu.py -q -x -k "all_gpus or three" > gpurun_out/mx.log 2>&1; echo "rc=$?" >> gpurun_out/mx.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $N --steps 500 > gpurun_out/x_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/x_n$N.log
