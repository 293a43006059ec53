set -u
mkdir -p gpurun_out/io7
run() { # cfg name env...
  c=$1; n=$2; shift; shift
  env "$@" timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2> gpurun_out/io7/${c}_$n.err | tail -n1 > gpurun_out/io7/${c}_$n.json
  python -c "import json; d=json.loads(open('gpurun_out/io7/${c}_$n.json').read()); print('$c $n', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
}
run c2 plain SF_NO_IO_OVERLAP=1
run c2 default SF_X=0
run c2 plain2 SF_NO_IO_OVERLAP=1
run c2 default2 SF_X=0
run c3o4 default SF_X=0
run c3o16 default SF_X=0
run c4 default SF_X=0
