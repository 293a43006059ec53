#!/bin/bash
# round-2 GPU check 4: parity of the decoupled queue kernels, A/B, ncu captures
mkdir -p gpurun_out/r2d
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variant or decoupled" > gpurun_out/r2d/parity.log 2>&1
echo "rc=$?" >> gpurun_out/r2d/parity.log
timeout 900 python tools/ab_time.py c3o12 8 "" "SF_VECQD=1" "SF_VECQD=2" > gpurun_out/r2d/ab_c3o12.jsonl 2>&1
timeout 900 python tools/ab_time.py c3o16 8 "" "SF_VECQD=1" "SF_VECQD=2" > gpurun_out/r2d/ab_c3o16.jsonl 2>&1
timeout 900 python tools/ab_time.py c3o8 10 "" "SF_VECQ=1" "SF_VECQ=1,SF_VECQD=1" "SF_VECQ=1,SF_VECQD=2" > gpurun_out/r2d/ab_c3o8.jsonl 2>&1
timeout 900 python tools/ab_time.py c4 4 "" "SF_VECQ=1" > gpurun_out/r2d/ab_c4.jsonl 2>&1
timeout 1200 python tools/ab_fwi.py 3 250 "" "SF_ZCHUNKS=2" "SF_ZCHUNKS=4" "SF_ZCHUNKS=6" > gpurun_out/r2d/ab_c5.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 200 --csv \
  --log-file gpurun_out/r2d/c4_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
  > gpurun_out/r2d/c4_launches.log 2>&1
tools/ncu_one.sh r2_vec_c4 c4 "acoustic3d_vec_kernel<4, true, 8"
tools/ncu_one.sh r2_vec_c5fwd c5 "acoustic3d_vec_kernel<4, true, 8"
tools/ncu_one.sh r2_vecgrad_c5 c5 "acoustic3d_vec_kernel<4, false, 4, true" 5
tools/ncu_one.sh r2_tb_c1 c1 "diffusion_tb"
tools/ncu_one.sh r2_vecq_c3o12 c3o12 "acoustic3d_vecq_kernel"
