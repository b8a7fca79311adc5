#!/bin/bash
# A/B of programmatic-dependent-launch masks at N = all visible GPUs (interleaved, 2 rounds).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for r in 1 2; do
for v in 0 15 13 9 5 12; do
  LMSGD_PDL_MASK=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$r bench.py --gpus $N --no-profile --steps 2000 > gpurun_out/ab_m${v}_r$r.log 2>&1
done
done
