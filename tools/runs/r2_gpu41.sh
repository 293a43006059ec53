set -u
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variant" 2>&1 | tail -2
timeout 900 python tools/ab_time.py c4 4 "SF_VEC_AQ2=0" "SF_VEC_AQ2=1" 2>&1 | grep -E "^\{" | tee -a gpurun_out/ab/ab8.jsonl
timeout 900 python tools/ab_time.py c3o8 8 "SF_VEC_AQ2=0" "SF_VEC_AQ2=1" 2>&1 | grep -E "^\{" | tee -a gpurun_out/ab/ab8.jsonl
