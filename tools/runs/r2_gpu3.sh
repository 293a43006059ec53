#!/bin/bash
# round-2 GPU check 3: parity of the changed vector kernels + the unrolled
# queue kernel, then A/B of the queue variants and the headline config
mkdir -p gpurun_out/r2c
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2c/parity.log 2>&1
echo "rc=$?" >> gpurun_out/r2c/parity.log
timeout 900 python tools/ab_time.py c3o16 8 "" "SF_VECQU=1" "SF_VECQU=1,SF_VEC_WARPS=8" > gpurun_out/r2c/ab_c3o16.jsonl 2>&1
timeout 900 python tools/ab_time.py c3o12 8 "" "SF_VECQU=1" "SF_VECQU=1,SF_VEC_WARPS=8" > gpurun_out/r2c/ab_c3o12.jsonl 2>&1
timeout 900 python tools/ab_time.py c4 5 "" > gpurun_out/r2c/ab_c4.jsonl 2>&1
timeout 900 python tools/ab_time.py c3o8 10 "" > gpurun_out/r2c/ab_c3o8.jsonl 2>&1
timeout 900 python tools/ab_time.py c2 20 "" > gpurun_out/r2c/ab_c2.jsonl 2>&1
