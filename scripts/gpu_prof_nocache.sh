#!/bin/bash
# Steady-state DRAM traffic of the k = 1 kernels (ncu without cache flushing between kernels).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SHORT="bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 --no-profile"
timeout 300 python $SHORT > gpurun_out/plain_nc.log 2>&1 && \
timeout 900 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum -k regex:"k_update|k_pack" -s 10 -c 6 --csv --log-file gpurun_out/nocache_guarded.csv python $SHORT > gpurun_out/ncu_nc.log 2>&1
timeout 300 python $SHORT --mode fused > gpurun_out/plain_nc2.log 2>&1 && \
timeout 900 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"k_fused1" -s 5 -c 3 --csv --log-file gpurun_out/nocache_fused.csv python $SHORT --mode fused > gpurun_out/ncu_nc2.log 2>&1
echo done
