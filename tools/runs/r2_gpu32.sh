set -u
mkdir -p gpurun_out/io5
run() { # cfg name env...
  c=$1; n=$2; shift; shift
  env "$@" timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2> gpurun_out/io5/${c}_$n.err | tail -n1 > gpurun_out/io5/${c}_$n.json
  python -c "import json; d=json.loads(open('gpurun_out/io5/${c}_$n.json').read()); print('$c $n', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
}
for c in c3o4 c3o8; do
run $c default SF_X=0
run $c z64 SF_IO_CHUNK_PLANES=64
run $c z64_k60_40 SF_IO_CHUNK_PLANES=64 SF_IO_STEPS=60 SF_IO_TAIL_STEPS=40
run $c z128_k60_40 SF_IO_STEPS=60 SF_IO_TAIL_STEPS=40
run $c z96 SF_IO_CHUNK_PLANES=96
done
run c4 z32 SF_IO_CHUNK_PLANES=32
run c4 z128 SF_IO_CHUNK_PLANES=128
run c4 k128_96 SF_IO_STEPS=128 SF_IO_TAIL_STEPS=96
run c4 k80_50 SF_IO_STEPS=80 SF_IO_TAIL_STEPS=50
