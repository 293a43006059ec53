#!/bin/bash
# Bench lines for every config (default = c4 with the CPU baseline), the
# reference arm, and the one-rank slab path -> gpurun_out/bench_all/
set -u
mkdir -p gpurun_out/bench_all
timeout 1200 python bench.py > gpurun_out/bench_all/c4.json 2> gpurun_out/bench_all/c4.err
for c in c1 c2 c3o4 c3o8 c3o12 c3o16 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_all/$c.json 2> gpurun_out/bench_all/$c.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_all/ref_c4.json 2> gpurun_out/bench_all/ref_c4.err
timeout 1200 python bench.py --force-slabs --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_all/slab1_c4.json 2> gpurun_out/bench_all/slab1_c4.err
tail -qn1 gpurun_out/bench_all/*.json | cut -c1-200
