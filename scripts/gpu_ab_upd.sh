#!/bin/bash
# A/B: register caps of the update kernels; N = 1 (k_update / k_fused1) and N = all GPUs (k_xupdate).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
run() {
  tag=$1; shift
  LMSGD_NVCC_EXTRA="$*" python paper_1711_04325_b200/build.py --force > /dev/null 2>&1
  timeout 300 python bench.py --steps 1000 --no-cpu-baseline > gpurun_out/abu_${tag}_n1.log 2>&1
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $N --steps 500 > gpurun_out/abu_${tag}_n$N.log 2>&1
  python - "$tag" "$N" <<'PY'
import json, sys
tag, n = sys.argv[1], sys.argv[2]
def last(f):
    l = [x for x in open(f) if x.startswith("{")]
    return json.loads(l[-1])
d1 = last(f"gpurun_out/abu_{tag}_n1.log"); dn = last(f"gpurun_out/abu_{tag}_n{n}.log")
t = dn["trace"]["us_median_per_rank"][0]
print(f"{tag}: N=1 step={d1['ms_per_step']*1e3:.1f} upd={d1['phases']['update']['us_per_launch']:.1f} fused={d1['variants']['fused_no_skip']['ms_per_step']*1e3:.1f} sgd={d1['variants']['sgd_phase']['ms_per_step']*1e3:.1f} | N={n} step={dn['ms_per_step']*1e3:.1f} upd={t['update']:.1f} sgd={dn['variants']['sgd_phase']['ms_per_step']*1e3:.1f} clk1={d1['clocks']['sm_mhz']} clkN={dn['clocks']['sm_mhz']}", flush=True)
PY
}
{
run base
run x6 -DLMSGD_XUPD_MINB=6
run x6f5u5 -DLMSGD_XUPD_MINB=6 -DLMSGD_FUSED_MINB=5 -DLMSGD_UPD_MINB=5
run x5 -DLMSGD_XUPD_MINB=5
run base2
} > gpurun_out/ab_upd.txt 2>&1
