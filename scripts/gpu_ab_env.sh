#!/bin/bash
# A/B of runtime knobs (environment) at N = all GPUs, one box. Args: tag=VAR=value ...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
python paper_1711_04325_b200/build.py > /dev/null 2>&1
for spec in "$@"; do
  tag=${spec%%=*}; kv=${spec#*=}
  env $kv timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $N --steps 500 --no-cpu-baseline > gpurun_out/abe_${tag}.log 2>&1
  python - "$tag" <<'PY'
import json, sys
v = sys.argv[1]
l = [x for x in open(f"gpurun_out/abe_{v}.log") if x.startswith("{")]
d = json.loads(l[-1]); t = d["trace"]["us_median_per_rank"][0]; nv = d["nvlink"]
print(f"{v}: ms={d['ms_per_step']*1e3:.1f}us p50={d['step_us_distribution']['median']:.1f} pack={t['pack']:.1f} wait={t['wait_all_packs']:.1f} red={t['reduce_block0']:.1f} fw={t['update_first_wait']:.1f} upd={t['update']:.1f} span={t['update_span']:.1f} xchg={nv['lmsgd_exchange_us']:.1f}", flush=True)
PY
done > gpurun_out/ab_env.txt 2>&1
