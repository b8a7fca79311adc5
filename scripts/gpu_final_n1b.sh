#!/bin/bash
# N = 1 with the out-of-place default: bench line (+ CPU baseline), R152 line, ncu launch
# list and full capture of k_fused1_oop (each ncu command after the plain run exited 0).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
python paper_1711_04325_b200/build.py > gpurun_out/final/build.log 2>&1
timeout 600 python bench.py > gpurun_out/final/n1.log 2>&1; echo "rc=$?" >> gpurun_out/final/n1.log
timeout 600 python bench.py --depth 152 --no-cpu-baseline > gpurun_out/final/n1_r152.log 2>&1; echo "rc=$?" >> gpurun_out/final/n1_r152.log
SHORT="bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3"
timeout 300 python $SHORT > gpurun_out/final/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_oop.csv python $SHORT > gpurun_out/final/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fused1_oop|k_repair1" -s 10 -c 2 -o gpurun_out/final/prof_oop python $SHORT > gpurun_out/final/ncu_full_oop.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_optim_gpu.py -q -x > gpurun_out/final/pt1.log 2>&1; echo "rc=$?" >> gpurun_out/final/pt1.log
