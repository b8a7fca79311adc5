#!/bin/bash
# GPU test suite only (single + multi-GPU tests at the box's GPU count)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python paper_1711_04325_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest ${PYTEST_ARGS:-tests} -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
