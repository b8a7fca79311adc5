#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python paper_1711_04325_b200/build.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "step_host or exchange" > gpurun_out/pe.log 2>&1; echo "rc=$?" >> gpurun_out/pe.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/e_n1.log 2>&1; echo "rc=$?" >> gpurun_out/e_n1.log
