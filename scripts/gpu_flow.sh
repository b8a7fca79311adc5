#!/bin/bash
# world > 1: parity of the pipelined flow exchange, then A/B flow vs two-kernel, traced.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
LMSGD_XFLOW=1 LMSGD_TIMEOUT_MS=10000 timeout 600 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/pytest_flow.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_flow.log
for r in 1 2; do
for v in 1 0; do
  LMSGD_XFLOW=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$r bench.py --gpus $N --steps 2000 > gpurun_out/flow_v${v}_r$r.log 2>&1
done
done
