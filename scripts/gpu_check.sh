#!/bin/bash
# One GPU round-trip: smoke, gpu tests, bench (guarded + fused), ncu launch list and
# full captures of the top kernels (each ncu command runs only after the same
# command exited 0 without ncu).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python bench.py --mode fused --no-cpu-baseline > gpurun_out/bench_fused.log 2>&1; echo "rc=$?" >> gpurun_out/bench_fused.log
SHORT="bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3"
timeout 300 python $SHORT > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python $SHORT > gpurun_out/ncu_launch.log 2>&1
timeout 300 python $SHORT > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_pack" -s 10 -c 2 -o gpurun_out/prof_guarded python $SHORT > gpurun_out/ncu_full.log 2>&1
timeout 300 python $SHORT --mode fused > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused1 -s 5 -c 1 -o gpurun_out/prof_fused python $SHORT --mode fused > gpurun_out/ncu_full_fused.log 2>&1
echo done
