#!/bin/bash
# NVLink peer-memory micro-benchmark (tools/p2pbench.cu) on a 2+ GPU box.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ./tools/p2pbench > gpurun_out/p2pbench.log 2>&1; echo "rc=$?" >> gpurun_out/p2pbench.log
timeout 300 ./tools/p2pbench 3194880 > gpurun_out/p2pbench_shard.log 2>&1; echo "rc=$?" >> gpurun_out/p2pbench_shard.log
