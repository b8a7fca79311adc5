#!/bin/bash
# Full validation on a 4-GPU box: all GPU tests, smoke, benches (N=1,4; R152), tiny-K runs.
cd $GRAFT_REPO_ROOT
bash scripts/gpu_multi.sh
bash scripts/gpu_smallk.sh
