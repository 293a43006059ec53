#!/bin/bash
mkdir -p gpurun_out/r2i
timeout 2400 python -m pytest tests/test_gpu_configs.py -m gpu -q -rA -k "full" --durations=0 > gpurun_out/r2i/full_loops.log 2>&1
echo "rc=$?" >> gpurun_out/r2i/full_loops.log
