#!/bin/bash
# Multi-GPU round-trip: all GPU tests (single + multi), smoke, bench at N=1 (guarded,
# fused) and at N = all GPUs (traced), plus the ResNet-152 buffer (config C5 sizes).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python paper_1711_04325_b200/build.py > gpurun_out/build.log 2>&1   # no-op unless a source is newer than the .so
N=$(nvidia-smi -L | wc -l)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_n1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n1.log
timeout 300 python bench.py --mode fused --no-cpu-baseline > gpurun_out/bench_n1_fused.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n1_fused.log
timeout 300 python bench.py --depth 152 --no-cpu-baseline --steps 1000 > gpurun_out/bench_r152_n1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_r152_n1.log
if [ "$N" -gt 1 ]; then
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29500 bench.py --gpus $N > gpurun_out/bench_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n$N.log
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29501 bench.py --gpus $N --depth 152 --steps 1000 > gpurun_out/bench_r152_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/bench_r152_n$N.log
fi
echo done
