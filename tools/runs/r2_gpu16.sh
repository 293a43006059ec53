#!/bin/bash
mkdir -p gpurun_out/r2p
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "autotune or variant" > gpurun_out/r2p/parity.log 2>&1
echo "rc=$?" >> gpurun_out/r2p/parity.log
