#!/bin/bash
mkdir -p gpurun_out/r2k
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variant or long_chunks" > gpurun_out/r2k/parity.log 2>&1
echo "rc=$?" >> gpurun_out/r2k/parity.log
timeout 900 python tools/ab_time.py c3o16 10 "" "SF_VECQ_FORM=tmem" > gpurun_out/r2k/ab_c3o16.jsonl 2>&1
timeout 900 python tools/ab_time.py c3o12 10 "" "SF_VECQ_FORM=tmem" > gpurun_out/r2k/ab_c3o12.jsonl 2>&1
