set -u
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "reciprocal or orders or parity or variant" > gpurun_out/ab/tests.log 2>&1; tail -3 gpurun_out/ab/tests.log
for c in c4 c3o8 c3o16 c3o12 c2; do
  r=8; [ $c = c4 ] && r=4
  timeout 900 python tools/ab_lib.py tools/_ab/base.so $c $r 2>&1 | grep -E "^\{" | tee -a gpurun_out/ab/ab1.jsonl
done
