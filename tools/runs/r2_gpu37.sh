set -u
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variant or fwi" > gpurun_out/ab/tests_aq8.log 2>&1; tail -2 gpurun_out/ab/tests_aq8.log
SF_VEC_AQ8=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_fwi_taylor.py -m gpu -x -q -k "fwi or taylor" 2>&1 | tail -2
timeout 900 python tools/ab_fwi.py 5 250 "SF_VEC_AQ8=0" "SF_VEC_AQ8=1" 2>&1 | grep -E "^\{" | tee -a gpurun_out/ab/ab7.jsonl
timeout 900 python tools/ab_time.py c3o8 8 "SF_VEC_WARPS=8,SF_VEC_AQ8=0" "SF_VEC_WARPS=8,SF_VEC_AQ8=1" "SF_VEC_WARPS=16" 2>&1 | grep -E "^\{" | tee -a gpurun_out/ab/ab7.jsonl
