#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python paper_1711_04325_b200/build.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "out_of_place or fused or k1" > gpurun_out/oop.log 2>&1; echo "rc=$?" >> gpurun_out/oop.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/oop_bench.log 2>&1; echo "rc=$?" >> gpurun_out/oop_bench.log
