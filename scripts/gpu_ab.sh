#!/bin/bash
# A/B: the previous commit's build (ab_old/) against the working tree, alternating on one box.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python paper_1711_04325_b200/build.py > gpurun_out/build.log 2>&1   # no-op unless a source is newer than the .so
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/ab_gpu.txt
for i in 1 2; do
  for v in new old; do
    d=.; [ $v = old ] && d=ab_old
    timeout 300 python $d/bench.py --no-cpu-baseline --no-profile >> gpurun_out/ab_n1_$v.log 2>&1
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600+i)) $d/bench.py --gpus 2 --no-profile >> gpurun_out/ab_n2_$v.log 2>&1
  done
done
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ab_pytest.log
