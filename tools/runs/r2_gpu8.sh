#!/bin/bash
# round-2 GPU check 8: full GPU suite, then every bench line
mkdir -p gpurun_out/r2h
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2h/gputest_all.log 2>&1
echo "rc=$?" >> gpurun_out/r2h/gputest_all.log
bash tools/bench_all.sh > gpurun_out/r2h/bench_all.txt 2>&1
