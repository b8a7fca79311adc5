#!/bin/bash
# compute-sanitizer memcheck (one tool per call) on the smoke test: k = 1 ctx step
# (pack + update), simulated k = 4 (pack x4, reduce, update).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_plain.log 2>&1 && \
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_memcheck.log 2>&1
echo "rc=$?" >> gpurun_out/sanitizer_memcheck.log
