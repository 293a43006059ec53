set -u
mkdir -p gpurun_out/io3
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/io3/tests_parity.log 2>&1; tail -3 gpurun_out/io3/tests_parity.log
for c in c4 c3o4 c3o8 c3o16 c2; do
for v in 0 1; do
  st=5; [ $c = c4 ] && st=3
  SF_NO_IO_OVERLAP=$v timeout 900 python bench.py --config $c --steps $st --warmup 2 --no-cpu-baseline 2> gpurun_out/io3/${c}_$v.err | tail -n1 > gpurun_out/io3/${c}_nooverlap$v.json
  python -c "import json,sys; d=json.loads(open('gpurun_out/io3/${c}_nooverlap$v.json').read()); print('$c no_overlap=$v', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done
done
