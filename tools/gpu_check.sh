#!/bin/bash
# One gpurun call: GPU parity tests, bench lines for the given configs, and an
# ncu launch-time list (per-launch kernel durations) for each config.
#   tools/gpu_check.sh "c2 c3o8 c3o16"   [TESTS=0 to skip pytest] [NCU=0]
set -u
CFGS=${1:-c2}
mkdir -p gpurun_out/chk
if [ "${TESTS:-1}" = 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/chk/gpu_tests.log 2>&1
  echo "tests_rc=$?" >> gpurun_out/chk/gpu_tests.log
  tail -3 gpurun_out/chk/gpu_tests.log
fi
for c in $CFGS; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/chk/bench_$c.log 2>&1
  tail -1 gpurun_out/chk/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'frac', round(d['roofline']['frac'],3), d['roofline'].get('kernel'), 'clk', d['clocks']['sm_mhz'])" 2>&1 | tail -1
done
if [ "${NCU:-1}" = 1 ]; then
  for c in $CFGS; do
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 60 --csv \
      --log-file gpurun_out/chk/launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
    python - "$c" <<'PY'
import csv, sys, collections
c = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/chk/launches_{c}.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
agg = collections.defaultdict(list)
for r in rows[1:]:
    v = float(r[vi].replace(",", "")); v = v / 1000 if r[ui] == "ns" else v * 1000 if r[ui] == "ms" else v
    agg[r[ki].split("(")[0]].append(v)
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    v.sort(); print(c, k[:70], len(v), "median_us", round(v[len(v)//2], 2))
PY
  done
fi
