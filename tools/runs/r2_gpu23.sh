set -u
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "last" > gpurun_out/ab/tests_last.log 2>&1; tail -3 gpurun_out/ab/tests_last.log
for c in c3o16 c3o12; do
timeout 900 python tools/ab_time.py $c 8 "SF_VECQ_FORM=pinned" "SF_VECQ_FORM=free" "SF_VECQ_FORM=last" 2>&1 | grep -E "^\{" | tee -a gpurun_out/ab/ab3.jsonl
done
