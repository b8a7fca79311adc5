#!/bin/bash
# One parameterised gpurun payload (run from the repo root on the GPU box):
#   gpurun --timeout S -- 'bash scripts/gpu.sh TASK [TASK ...]'
# TASKs (run in order, each logged to gpurun_out/<task>.log with its rc):
#   tests       pytest -m gpu (every GPU test at this box's GPU count; PYTEST_ARGS overrides the target)
#   smoke       __graft_entry__.smoke()
#   bench1      bench.py at N = 1 (BENCH_ARGS appended)
#   benchN      bench.py at N = 2, 4, 8 (each N <= the box's GPU count; BENCH_ARGS appended)
#   ref         bench.py --impl reference at N = 1
#   launches    ncu launch list of a short N = 1 bench (gpu__time_duration, no clock control)
#   ncufull     ncu --set full of the N = 1 dominant kernel (NCU_KERNEL regex, default k_fused1_oop)
#   ab          A/B: ab_old/ (an older tree) against this one, alternating, N = 1 and N = all
#   cmd         eval "$CMD" (anything else)
cd "${GRAFT_REPO_ROOT:-.}" || exit 1
mkdir -p gpurun_out
python paper_1711_04325_b200/build.py > gpurun_out/build.log 2>&1 || { echo "build failed"; exit 1; }
N=$(nvidia-smi -L | wc -l)
run() {   # run NAME TIMEOUT CMD...
  local name=$1 to=$2; shift 2
  timeout "$to" "$@" > "gpurun_out/$name.log" 2>&1
  echo "rc=$?" >> "gpurun_out/$name.log"
  tail -2 "gpurun_out/$name.log"
}
tr() { echo python -m torch.distributed.run --nnodes=1 --nproc-per-node "$1" --master-addr 127.0.0.1 --master-port "$2"; }
for task in "$@"; do
  case $task in
    tests) run pytest_gpu 1500 python -m pytest ${PYTEST_ARGS:-tests} -m gpu -q -rs --timeout 900 --durations=15 ;;
    smoke) run smoke 300 python -c "import __graft_entry__ as g; g.smoke()" ;;
    bench1) run bench_n1 600 python bench.py $BENCH_ARGS ;;
    benchN) for n in 2 4 8; do
              [ "$N" -ge "$n" ] && run "bench_n$n" 600 $(tr $n $((29500 + n))) bench.py --gpus $n $BENCH_ARGS
            done ;;
    ref) run bench_ref 600 python bench.py --impl reference --steps 3 --warmup 3 ;;
    launches) run ncu_launches 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
                --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline ;;
    ncufull) run ncu_full 900 ncu --set full --clock-control none --import-source on \
               -k "regex:${NCU_KERNEL:-k_fused1_oop}" -s 5 -c 1 -o gpurun_out/full -f \
               python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-profile ;;
    ab) for i in 1 2; do
          for v in new old; do
            d=.; [ $v = old ] && d=ab_old
            run "ab_n1_${v}_$i" 300 python $d/bench.py --no-cpu-baseline --no-profile $BENCH_ARGS
            [ "$N" -ge 2 ] && run "ab_n${N}_${v}_$i" 300 $(tr $N $((29600 + i))) $d/bench.py --gpus $N --no-profile $BENCH_ARGS
          done
        done ;;
    cmd) run cmd 3000 bash -c "$CMD" ;;
    *) echo "unknown task $task" ;;
  esac
done
echo done
