#!/bin/bash
# Multi-GPU parity worker on every GPU of the box (+ k = 3 when >= 3 GPUs).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python paper_1711_04325_b200/build.py > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/mt.log 2>&1; echo "rc=$?" >> gpurun_out/mt.log
