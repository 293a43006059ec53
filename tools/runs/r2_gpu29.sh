set -u
mkdir -p gpurun_out/io2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "overlapped" > gpurun_out/io2/tests_overlap.log 2>&1; tail -5 gpurun_out/io2/tests_overlap.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/io2/tests_parity.log 2>&1; tail -3 gpurun_out/io2/tests_parity.log
for v in 0 1; do
  SF_NO_IO_OVERLAP=$v timeout 900 python bench.py --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/io2/c4_nooverlap$v.json 2> gpurun_out/io2/c4_nooverlap$v.err
  tail -n1 gpurun_out/io2/c4_nooverlap$v.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('no_overlap=$v', round(d['value'],1), 'e2e', d['e2e'])"
done
SF_IO_TAIL_STEPS=0 timeout 900 python bench.py --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/io2/c4_tail0.json 2> gpurun_out/io2/c4_tail0.err
tail -n1 gpurun_out/io2/c4_tail0.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tail0', round(d['value'],1), 'e2e', d['e2e'])"
timeout 900 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline | tail -n1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', round(d['value'],1), 'e2e', d['e2e'])"
SF_NO_IO_OVERLAP=1 timeout 900 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline | tail -n1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 no overlap', round(d['value'],1), 'e2e', d['e2e'])"
