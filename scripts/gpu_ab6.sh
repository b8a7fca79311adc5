#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for r in 1 2; do
for v in 1 5; do
  LMSGD_PDL_MASK=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$r bench.py --gpus $N > gpurun_out/ab6_m${v}_r$r.log 2>&1
done
done
