#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ./tools/xbench > gpurun_out/xbench.log 2>&1; echo "rc=$?" >> gpurun_out/xbench.log
