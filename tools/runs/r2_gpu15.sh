#!/bin/bash
mkdir -p gpurun_out/r2o
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variant" > gpurun_out/r2o/parity.log 2>&1
echo "rc=$?" >> gpurun_out/r2o/parity.log
timeout 900 python tools/ab_time.py c2 20 "" "SF_VEC_NX=1,SF_VEC_WARPS=8" "SF_VEC_NX=2,SF_VEC_WARPS=8" > gpurun_out/r2o/ab_c2.jsonl 2>&1
timeout 900 python tools/ab_time.py c3o4 10 "" "SF_VEC_WARPS=8" "SF_VEC_NX=1,SF_VEC_WARPS=8" > gpurun_out/r2o/ab_c3o4.jsonl 2>&1
timeout 1500 python tools/ab_fwi.py 3 1000 "" > gpurun_out/r2o/fwi_nt1000.jsonl 2>&1
timeout 900 python tools/ab_fwi.py 3 250 "" > gpurun_out/r2o/fwi_nt250.jsonl 2>&1
