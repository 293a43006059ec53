#!/bin/bash
# round-2 GPU check 7: in-process A/B of the round-1 and round-2 queue kernels
mkdir -p gpurun_out/r2g
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variant and (12 or 16)" > gpurun_out/r2g/parity.log 2>&1
echo "rc=$?" >> gpurun_out/r2g/parity.log
timeout 900 python tools/ab_time.py c3o12 10 "" "SF_VECQ_R1=1" > gpurun_out/r2g/ab_c3o12.jsonl 2>&1
timeout 900 python tools/ab_time.py c3o16 10 "" "SF_VECQ_R1=1" > gpurun_out/r2g/ab_c3o16.jsonl 2>&1
