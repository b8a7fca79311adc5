#!/bin/bash
# world > 1: parity of the one-kernel step, then A/B (one kernel vs three kernels) at N = all GPUs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
LMSGD_TIMEOUT_MS=10000 timeout 600 python -m pytest tests/test_multigpu.py -q > gpurun_out/pytest_mgpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_mgpu.log
for r in 1 2; do
for v in 1 0; do
  LMSGD_XSTEP=$v timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$r bench.py --gpus $N --no-profile --steps 2000 > gpurun_out/xs_v${v}_r$r.log 2>&1
done
done
LMSGD_XSTEP=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29539 bench.py --gpus $N --trace --steps 1000 > gpurun_out/xs_trace.log 2>&1
