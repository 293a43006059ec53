set -u
mkdir -p gpurun_out/io6
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "overlapped" > gpurun_out/io6/tests_overlap.log 2>&1; tail -2 gpurun_out/io6/tests_overlap.log
run() { # cfg name env...
  c=$1; n=$2; shift; shift
  env "$@" timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2> gpurun_out/io6/${c}_$n.err | tail -n1 > gpurun_out/io6/${c}_$n.json
  python -c "import json; d=json.loads(open('gpurun_out/io6/${c}_$n.json').read()); print('$c $n', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
}
run c2 plain SF_NO_IO_OVERLAP=1
run c2 z96_k60_40 SF_IO_OVERLAP=1 SF_IO_CHUNK_PLANES=96 SF_IO_STEPS=60 SF_IO_TAIL_STEPS=40
run c2 z64_k60_40 SF_IO_OVERLAP=1 SF_IO_CHUNK_PLANES=64 SF_IO_STEPS=60 SF_IO_TAIL_STEPS=40
run c3o4 default SF_X=0
run c3o8 default SF_X=0
run c4 default SF_X=0
