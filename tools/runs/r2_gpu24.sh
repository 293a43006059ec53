set -u
mkdir -p gpurun_out/ab
for c in c3o10 c3o14 c3o12 c3o16; do
timeout 900 python tools/ab_time.py $c 10 "SF_VECQ_FORM=pinned" "SF_VECQ_FORM=free" "SF_VECQ_FORM=last" 2>&1 | grep -E "^\{" | tee -a gpurun_out/ab/ab4.jsonl
done
