#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 ./tools/flagbench > gpurun_out/flagbench.log 2>&1; echo "rc=$?" >> gpurun_out/flagbench.log
