#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 600 env LMSGD_PDL_MASK=3 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/pytest_mgpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mgpu.log
for r in 1 2; do
for v in 1 3; do
  LMSGD_PDL_MASK=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$r bench.py --gpus $N --no-profile > gpurun_out/ab5_m${v}_r$r.log 2>&1
done
done
