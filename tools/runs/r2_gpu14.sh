#!/bin/bash
mkdir -p gpurun_out/r2n
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "fwi" > gpurun_out/r2n/parity.log 2>&1
echo "rc=$?" >> gpurun_out/r2n/parity.log
timeout 1500 python tools/ab_fwi.py 4 250 "" "SF_VEC_WARPS=16" > gpurun_out/r2n/ab_c5.jsonl 2>&1
