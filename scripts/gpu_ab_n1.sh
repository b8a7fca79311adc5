#!/bin/bash
# A/B of compile-time knobs at N = 1 (bench headline), one box. Args: tag=flags ...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for spec in "$@"; do
  tag=${spec%%=*}; flags=${spec#*=}
  LMSGD_NVCC_EXTRA="$flags" python paper_1711_04325_b200/build.py --force > /dev/null 2>&1
  timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab1_${tag}.log 2>&1
  python - "$tag" <<'PY'
import json, sys
v = sys.argv[1]
l = [x for x in open(f"gpurun_out/ab1_{v}.log") if x.startswith("{")]
d = json.loads(l[-1])
print(f"{v}: ms={d['ms_per_step']*1e3:.1f}us p50={d['step_us_distribution']['median']:.1f} prof={d['phases']['pack']['us_per_launch']:.1f} inplace={d['variants']['guarded_in_place']['ms_per_step']*1e3:.1f} clk={d['clocks']['sm_mhz']} {d['clocks']['reasons']}", flush=True)
PY
done > gpurun_out/ab_n1.txt 2>&1
python paper_1711_04325_b200/build.py --force > /dev/null 2>&1
