#!/bin/bash
# Final single-GPU evidence: headline bench (default), fused and R152 lines, the
# reference arm, then the ncu launch list and full captures (each ncu command only
# after the same command exited 0 without ncu).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
python paper_1711_04325_b200/build.py > gpurun_out/final/build.log 2>&1
timeout 600 python bench.py > gpurun_out/final/n1.log 2>&1; echo "rc=$?" >> gpurun_out/final/n1.log
timeout 600 python bench.py --mode fused --no-cpu-baseline > gpurun_out/final/n1_fused.log 2>&1; echo "rc=$?" >> gpurun_out/final/n1_fused.log
timeout 600 python bench.py --depth 152 --no-cpu-baseline > gpurun_out/final/n1_r152.log 2>&1; echo "rc=$?" >> gpurun_out/final/n1_r152.log
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/final/ref_n1.log 2>&1; echo "rc=$?" >> gpurun_out/final/ref_n1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final/smoke.log
SHORT="bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3"
timeout 300 python $SHORT > gpurun_out/final/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches.csv python $SHORT > gpurun_out/final/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_pack" -s 10 -c 2 -o gpurun_out/final/prof_guarded python $SHORT > gpurun_out/final/ncu_full.log 2>&1
timeout 300 python $SHORT --mode fused > gpurun_out/final/plain_f.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused1 -s 5 -c 1 -o gpurun_out/final/prof_fused python $SHORT --mode fused > gpurun_out/final/ncu_full_fused.log 2>&1
echo done > gpurun_out/final/done.txt
