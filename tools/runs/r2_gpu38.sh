set -u
mkdir -p gpurun_out/last
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/last/gpu_tests.log 2>&1; tail -2 gpurun_out/last/gpu_tests.log
timeout 900 python bench.py > gpurun_out/last/c4.json 2> gpurun_out/last/c4.err; tail -n1 gpurun_out/last/c4.json | cut -c1-160
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline 2> gpurun_out/last/c5.err | tail -n1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', round(d['value'],1), d['e2e'])"
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline 2> gpurun_out/last/c1.err | tail -n1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c1', round(d['value'],1), d['clocks'])"
