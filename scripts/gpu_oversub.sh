#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python paper_1711_04325_b200/build.py > gpurun_out/build.log 2>&1
timeout 1000 python -m pytest tests/test_multigpu.py -q -x -k world8 --durations=1 > gpurun_out/ov.log 2>&1; echo "rc=$?" >> gpurun_out/ov.log
