#!/bin/bash
# round-2 GPU check 1: smoke, new medium + config-layout tests, then the default bench
mkdir -p gpurun_out/r2a
(nvidia-smi; lscpu | head -20; nproc) > gpurun_out/r2a/machine.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r2a/smoke.log
timeout 2400 python -m pytest tests/test_medium.py tests/test_gpu_configs.py tests/test_fwi_taylor.py -m gpu -q -rA --timeout 1200 > gpurun_out/r2a/tests_new.log 2>&1
echo "rc=$?" >> gpurun_out/r2a/tests_new.log
timeout 900 python bench.py > gpurun_out/r2a/bench_c4.json 2> gpurun_out/r2a/bench_c4.err
echo "rc=$?" >> gpurun_out/r2a/bench_c4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2a/ref_c4.json 2> gpurun_out/r2a/ref_c4.err
echo "rc=$?" >> gpurun_out/r2a/ref_c4.err
