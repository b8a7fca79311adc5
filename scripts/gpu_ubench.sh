#!/bin/bash
# Kernel-variant micro-benchmark on one B200 (tools/ubench.cu).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ./tools/ubench > gpurun_out/ubench.log 2>&1; echo "rc=$?" >> gpurun_out/ubench.log
timeout 300 ./tools/ubench 1000003 > gpurun_out/ubench_small.log 2>&1; echo "rc=$?" >> gpurun_out/ubench_small.log
