#!/bin/bash
# A/B of two kernels.cu versions on one box (abtmp/kernels_{new,old}.cu, untracked):
# bench N = all GPUs, alternating builds; then the GPU tests with the new version.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for V in new old new old; do
  cp abtmp/kernels_$V.cu paper_1711_04325_b200/csrc/kernels.cu
  python paper_1711_04325_b200/build.py --force > /dev/null 2>&1
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $N --steps 500 --no-cpu-baseline > gpurun_out/abs_${V}.log 2>&1
  python - "$V" <<'PY'
import json, sys
v = sys.argv[1]
l = [x for x in open(f"gpurun_out/abs_{v}.log") if x.startswith("{")]
d = json.loads(l[-1]); t = d["trace"]["us_median_per_rank"][0]; nv = d["nvlink"]
print(f"{v}: bn={d["bn_stats_allreduce"]["us_per_call"]:.1f} ms={d["ms_per_step"]*1e3:.1f}us p50={d['step_us_distribution']['median']:.1f} pack={t['pack']:.1f} wait={t['wait_all_packs']:.1f} red={t['reduce_block0']:.1f} fw={t['update_first_wait']:.1f} upd={t['update']:.1f} xchg={nv['lmsgd_exchange_us']:.1f} nccl={nv['nccl_fp16_allreduce_us']:.1f} sgd={d['variants']['sgd_phase']['ms_per_step']*1e3:.1f}", flush=True)
PY
done > gpurun_out/ab_src.txt 2>&1
cp abtmp/kernels_new.cu paper_1711_04325_b200/csrc/kernels.cu
python paper_1711_04325_b200/build.py --force > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_multigpu.py tests/test_gpu_parity.py -q -x > gpurun_out/abs_tests.log 2>&1; echo "rc=$?" >> gpurun_out/abs_tests.log
