#!/bin/bash
mkdir -p gpurun_out/r2m
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2m/gputest_all.log 2>&1
echo "rc=$?" >> gpurun_out/r2m/gputest_all.log
timeout 1200 python bench.py > gpurun_out/r2m/c4.json 2> gpurun_out/r2m/c4.err
timeout 900 python bench.py --config c3o8 --steps 5 --warmup 3 > gpurun_out/r2m/c3o8.json 2> gpurun_out/r2m/c3o8.err
timeout 1200 python bench.py --force-slabs --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2m/slab1_c4.json 2> gpurun_out/r2m/slab1_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 200 --csv \
  --log-file gpurun_out/r2m/c4_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
  > gpurun_out/r2m/c4_launches.log 2>&1
tools/ncu_one.sh r2_vec16_c4 c4 "acoustic3d_vec_kernel<.int.4, .bool.1, .int.16"
