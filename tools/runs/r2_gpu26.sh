set -u
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variant and (WARPS=8 or WARPS=12)" > gpurun_out/ab/tests_w.log 2>&1; tail -3 gpurun_out/ab/tests_w.log
for c in c3o16 c3o14; do
timeout 900 python tools/ab_time.py $c 8 "SF_VECQ_FORM=pinned" "SF_VEC_WARPS=8" "SF_VEC_WARPS=8,SF_VECQ_FORM=last" "SF_VEC_WARPS=12" "SF_VEC_WARPS=12,SF_VECQ_FORM=last" "SF_VEC_WARPS=12,SF_VECQ_FORM=last,SF_TMA_STAGES=4" 2>&1 | grep -E "^\{" | tee -a gpurun_out/ab/ab5.jsonl
done
for c in c3o12 c3o10; do
timeout 900 python tools/ab_time.py $c 8 "SF_VECQ_FORM=pinned" "SF_VECQ_FORM=last" "SF_VEC_WARPS=8,SF_VECQ_FORM=pinned" "SF_VEC_WARPS=8,SF_VECQ_FORM=last" "SF_VEC_WARPS=8,SF_VECQ_FORM=last,SF_TMA_STAGES=4" 2>&1 | grep -E "^\{" | tee -a gpurun_out/ab/ab5.jsonl
done
