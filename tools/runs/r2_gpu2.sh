#!/bin/bash
# round-2 GPU check 2: acceptance via sf-cuda-cc, Taylor test, knob A/B on the
# headline and high-order kernels, the full GPU suite
mkdir -p gpurun_out/r2b
timeout 1500 python -m pytest tests/test_acceptance_gpu.py tests/test_fwi_taylor.py -m gpu -q -rA > gpurun_out/r2b/tests_new.log 2>&1
echo "rc=$?" >> gpurun_out/r2b/tests_new.log
timeout 900 python tools/ab_time.py c4 5 "" "SF_VEC_RPL=2" "SF_TMA_STAGES=2" "SF_TMA_STAGES=4" > gpurun_out/r2b/ab_c4.jsonl 2>&1
timeout 900 python tools/ab_time.py c3o16 8 "" "SF_VEC_WARPS=8" "SF_TMA_STAGES=2" "SF_TMA_STAGES=4" "SF_VECQ2=1" > gpurun_out/r2b/ab_c3o16.jsonl 2>&1
timeout 900 python tools/ab_time.py c3o12 8 "" "SF_VEC_WARPS=8" "SF_TMA_STAGES=2" "SF_TMA_STAGES=4" "SF_VECQ2=1" > gpurun_out/r2b/ab_c3o12.jsonl 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --deselect tests/test_acceptance_gpu.py --deselect tests/test_fwi_taylor.py > gpurun_out/r2b/gputest_all.log 2>&1
echo "rc=$?" >> gpurun_out/r2b/gputest_all.log
