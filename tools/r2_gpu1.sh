#!/bin/bash
# round-2 GPU check 1: new medium + config-layout tests, then the default bench
mkdir -p gpurun_out/r2a
timeout 2400 python -m pytest tests/test_medium.py tests/test_gpu_configs.py -m gpu -x -q -rA > gpurun_out/r2a/tests_new.log 2>&1
echo "rc=$?" >> gpurun_out/r2a/tests_new.log
timeout 900 python bench.py > gpurun_out/r2a/bench_c4.json 2> gpurun_out/r2a/bench_c4.err
echo "rc=$?" >> gpurun_out/r2a/bench_c4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2a/ref_c4.json 2> gpurun_out/r2a/ref_c4.err
echo "rc=$?" >> gpurun_out/r2a/ref_c4.err
