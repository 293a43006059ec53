set -u
mkdir -p gpurun_out/io4
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "overlapped" > gpurun_out/io4/tests_overlap.log 2>&1; tail -2 gpurun_out/io4/tests_overlap.log
run() { # name env...
  n=$1; shift
  env "$@" timeout 600 python bench.py --config c2 --steps 5 --warmup 3 --no-cpu-baseline 2> gpurun_out/io4/$n.err | tail -n1 > gpurun_out/io4/$n.json
  python -c "import json; d=json.loads(open('gpurun_out/io4/$n.json').read()); print('$n', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
}
run plain SF_NO_IO_OVERLAP=1
run z32 SF_IO_OVERLAP=1 SF_IO_CHUNK_PLANES=32
run z64 SF_IO_OVERLAP=1 SF_IO_CHUNK_PLANES=64
run z96 SF_IO_OVERLAP=1 SF_IO_CHUNK_PLANES=96
run z64_k60_40 SF_IO_OVERLAP=1 SF_IO_CHUNK_PLANES=64 SF_IO_STEPS=60 SF_IO_TAIL_STEPS=40
run z96_k60_40 SF_IO_OVERLAP=1 SF_IO_CHUNK_PLANES=96 SF_IO_STEPS=60 SF_IO_TAIL_STEPS=40
