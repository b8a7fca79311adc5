#!/bin/bash
# k_pack on all 2^32 fp32 bit patterns vs the oracle codec (opt-in test, ~10 min).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python paper_1711_04325_b200/build.py > gpurun_out/build.log 2>&1
LMSGD_EXHAUSTIVE=1 timeout 1500 python -m pytest tests/test_gpu_parity.py -q -k all_fp32_patterns --durations=1 > gpurun_out/exhaustive.log 2>&1; echo "rc=$?" >> gpurun_out/exhaustive.log
