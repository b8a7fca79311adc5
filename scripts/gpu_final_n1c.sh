#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
python paper_1711_04325_b200/build.py > gpurun_out/final/build.log 2>&1
timeout 600 python bench.py > gpurun_out/final/n1.log 2>&1; echo "rc=$?" >> gpurun_out/final/n1.log
SHORT="bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3"
timeout 300 python $SHORT > gpurun_out/final/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_oop.csv python $SHORT > gpurun_out/final/ncu_launch.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final/smoke.log
