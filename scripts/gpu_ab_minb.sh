#!/bin/bash
# A/B: k_xstep1 register cap (min blocks/SM) at N = all GPUs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
for MB in 1 8 6 1; do
  LMSGD_NVCC_EXTRA="-DLMSGD_XSTEP_MINB=$MB" python paper_1711_04325_b200/build.py --force > /dev/null 2>&1
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $N --steps 500 > gpurun_out/ab_mb${MB}_n$N.log 2>&1
  python - "$MB" "$N" <<'PY'
import json, sys
mb, n = sys.argv[1], sys.argv[2]
l = [x for x in open(f"gpurun_out/ab_mb{mb}_n{n}.log") if x.startswith("{")]
d = json.loads(l[-1]); t = d["trace"]["us_median_per_rank"][0]; nv = d["nvlink"]
print(f"MB={mb} N={n} ms={d['ms_per_step']*1e3:.1f}us pack={t['pack']:.1f} wait={t['wait_all_packs']:.1f} red={t['reduce_block0']:.1f} fw={t['update_first_wait']:.1f} upd={t['update']:.1f} xchg={nv['lmsgd_exchange_us']:.1f} nccl={nv['nccl_fp16_allreduce_us']:.1f} sgd={d['variants']['sgd_phase']['ms_per_step']*1e3:.1f}", flush=True)
PY
done > gpurun_out/ab_minb.txt 2>&1
