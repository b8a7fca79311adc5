#!/bin/bash
# World-2 fold path: multi-GPU parity suite (fold on by default), then A/B bench lines.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python paper_1711_04325_b200/build.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -q -x -k "all_gpus or timeout" > gpurun_out/fold_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fold_tests.log
for F in 1 0 1 0; do
  LMSGD_FOLD2=$F timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 2 --steps 1000 --no-cpu-baseline > gpurun_out/fold_$F.log 2>&1
  python - "$F" <<'PY'
import json, sys
v = sys.argv[1]
l = [x for x in open(f"gpurun_out/fold_{v}.log") if x.startswith("{")]
d = json.loads(l[-1]); t = d["trace"]["us_median_per_rank"][0]; nv = d["nvlink"]
print(f"fold={v}: ms={d['ms_per_step']*1e3:.1f}us p50={d['step_us_distribution']['median']:.1f} pack={t['pack']:.1f} wait={t['wait_all_packs']:.1f} red={t['reduce_block0']:.1f} fw={t['update_first_wait']:.1f} upd={t['update']:.1f} span={t['update_span']:.1f} sgd={d['variants']['sgd_phase']['ms_per_step']*1e3:.1f}", flush=True)
PY
done > gpurun_out/ab_fold.txt 2>&1
