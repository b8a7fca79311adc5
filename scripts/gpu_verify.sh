#!/bin/bash
# Fresh-box check of the restored tree: build, GPU tests, smoke, N=1 and N=all bench lines.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
python paper_1711_04325_b200/build.py > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/v_n1.log 2>&1; echo "rc=$?" >> gpurun_out/v_n1.log
if [ $N -gt 1 ]; then
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $N > gpurun_out/v_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/v_n$N.log
fi
