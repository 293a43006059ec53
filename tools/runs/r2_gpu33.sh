set -u
mkdir -p gpurun_out/ab
timeout 900 python tools/ab_time.py c3o12 10 "SF_VECQ_FORM=last" "SF_VECQ_FORM=last,SF_TMA_STAGES=4" "SF_VECQ_FORM=last,SF_TMA_STAGES=2" 2>&1 | grep -E "^\{" | tee -a gpurun_out/ab/ab6.jsonl
timeout 900 python tools/ab_time.py c3o10 10 "SF_VECQ_FORM=pinned" "SF_VECQ_FORM=last,SF_TMA_STAGES=4" "SF_VECQ_FORM=pinned,SF_TMA_STAGES=4" 2>&1 | grep -E "^\{" | tee -a gpurun_out/ab/ab6.jsonl
timeout 900 python tools/ab_time.py c3o16 10 "SF_VECQ_FORM=pinned" "SF_VECQ_FORM=last,SF_TMA_STAGES=4" "SF_VECQ_FORM=pinned,SF_TMA_STAGES=4" 2>&1 | grep -E "^\{" | tee -a gpurun_out/ab/ab6.jsonl
