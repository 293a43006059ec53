#!/bin/bash
# Round-end style validation on one B200: smoke, GPU tests, bench lines for
# every config + reference arm + one-rank slab path, c2 launch list.
set -u
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke_rc=$?" >> gpurun_out/final/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final/gpu_tests.log 2>&1; echo "tests_rc=$?" >> gpurun_out/final/gpu_tests.log
tail -2 gpurun_out/final/gpu_tests.log; tail -2 gpurun_out/final/smoke.log
bash tools/bench_all.sh
cp -r gpurun_out/bench_all gpurun_out/final/
