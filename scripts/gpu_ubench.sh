#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ./tools/ubench > gpurun_out/ubench.txt 2>&1; echo "rc=$?" >> gpurun_out/ubench.txt
