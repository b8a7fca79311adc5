#!/bin/bash
# Single GPU: kernel micro-benchmark, then ncu launch list + full captures of the
# production kernels (each ncu command only after the same command exited 0).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 ./tools/ubench > gpurun_out/ubench.log 2>&1; echo "rc=$?" >> gpurun_out/ubench.log
SHORT="bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3"
timeout 300 python $SHORT > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python $SHORT > gpurun_out/ncu_launch.log 2>&1
timeout 300 python $SHORT > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_pack" -s 10 -c 2 -o gpurun_out/prof_guarded python $SHORT > gpurun_out/ncu_full.log 2>&1
timeout 300 python $SHORT --mode fused > gpurun_out/plain3.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fused.csv python $SHORT --mode fused > gpurun_out/ncu_launch_fused.log 2>&1
timeout 300 python $SHORT --mode fused > gpurun_out/plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused1 -s 5 -c 1 -o gpurun_out/prof_fused python $SHORT --mode fused > gpurun_out/ncu_full_fused.log 2>&1
echo done
