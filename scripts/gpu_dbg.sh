#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 tools/debug_wd.py > gpurun_out/dbg.log 2>&1; echo "rc=$?" >> gpurun_out/dbg.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29622 bench.py --gpus 2 --no-profile > gpurun_out/dbg_bench2.log 2>&1
timeout 300 python bench.py --no-profile --no-cpu-baseline > gpurun_out/dbg_bench1.log 2>&1
