#!/bin/bash
mkdir -p gpurun_out/r2q
timeout 1500 python tools/ab_fwi.py 4 250 "" "SF_VEC_WARPS=4" "SF_TMA_STAGES=4" "SF_TMA_STAGES_GRAD=5" > gpurun_out/r2q/ab_c5.jsonl 2>&1
