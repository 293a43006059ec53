#!/bin/bash
# Bench lines for every config (default = c2 with the CPU baseline), the
# reference arm, and the one-rank slab path -> gpurun_out/bench_all/
set -u
mkdir -p gpurun_out/bench_all
python bench.py > gpurun_out/bench_all/c2.json 2> gpurun_out/bench_all/c2.err
for c in c1 c3o4 c3o8 c3o12 c3o16 c4 c5; do
  python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_all/$c.json 2> gpurun_out/bench_all/$c.err
done
python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_all/ref_c2.json 2> gpurun_out/bench_all/ref_c2.err
python bench.py --force-slabs --steps 5 --warmup 3 > gpurun_out/bench_all/slab1.json 2> gpurun_out/bench_all/slab1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 50 -c 400 --csv \
  --log-file gpurun_out/bench_all/c2_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
tail -qn1 gpurun_out/bench_all/*.json | cut -c1-200
