#!/bin/bash
mkdir -p gpurun_out/r2l
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variant" > gpurun_out/r2l/parity.log 2>&1
echo "rc=$?" >> gpurun_out/r2l/parity.log
timeout 1200 python tools/ab_time.py c4 5 "" "SF_VEC_WARPS=16" > gpurun_out/r2l/ab_c4.jsonl 2>&1
timeout 900 python tools/ab_time.py c3o8 10 "" "SF_VEC_WARPS=16" > gpurun_out/r2l/ab_c3o8.jsonl 2>&1
