#!/bin/bash
# round-2 GPU check 2: pipe probe, new tests, full GPU suite, ncu captures
mkdir -p gpurun_out/r2b gpurun_out/prof
./tools/pipe_probe > gpurun_out/r2b/pipe.jsonl 2>&1
timeout 1500 python -m pytest tests/test_gpu_configs.py::test_c4_two_slab_chain_vs_port tests/test_fwi_taylor.py -m gpu -x -q -rA > gpurun_out/r2b/tests_new.log 2>&1
echo "rc=$?" >> gpurun_out/r2b/tests_new.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 200 --csv \
  --log-file gpurun_out/r2b/c4_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
  > gpurun_out/r2b/c4_launches.log 2>&1
KREGEX=acoustic3d_vec tools/ncu_full.sh "r2_vec_c4:c4 r2_vecq_c3o12:c3o12 r2_vec_c5fwd:c5"
KREGEX=diffusion_tb tools/ncu_full.sh "r2_tb_c1:c1"
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2b/gputest_all.log 2>&1
echo "rc=$?" >> gpurun_out/r2b/gputest_all.log
