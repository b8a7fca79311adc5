#!/bin/bash
# bench.py at N = all visible GPUs (and N=1 for reference), no tests.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_n1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n1.log
timeout 300 python bench.py --mode fused --no-cpu-baseline > gpurun_out/bench_n1_fused.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n1_fused.log
for n in 2 4 8; do
  if [ "$N" -ge "$n" ]; then
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$n bench.py --gpus $n > gpurun_out/bench_n$n.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n$n.log
  fi
done
echo done
