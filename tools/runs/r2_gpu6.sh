#!/bin/bash
# round-2 GPU check 6: balanced single-wave schedule for the queue kernel
mkdir -p gpurun_out/r2f
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -m gpu -q -x > gpurun_out/r2f/parity.log 2>&1
echo "rc=$?" >> gpurun_out/r2f/parity.log
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -k "c3" >> gpurun_out/r2f/parity.log 2>&1
echo "rc=$?" >> gpurun_out/r2f/parity.log
timeout 900 python tools/ab_time.py c3o12 8 "" "SF_NO_BALANCE=1" > gpurun_out/r2f/ab_c3o12.jsonl 2>&1
timeout 900 python tools/ab_time.py c3o16 8 "" "SF_NO_BALANCE=1" > gpurun_out/r2f/ab_c3o16.jsonl 2>&1
timeout 1200 python bench.py --config c4 --force-slabs --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r2f/slab_c4.json 2> gpurun_out/r2f/slab_c4.err
