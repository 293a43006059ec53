#!/bin/bash
# round-2 GPU check 5: queue kernel with pinned loop state, binding, slab C4, ncu
mkdir -p gpurun_out/r2e
free -g > gpurun_out/r2e/free.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_integration_binding.py -m gpu -q -x -k "variant or long_chunks or binding or c3" > gpurun_out/r2e/parity.log 2>&1
echo "rc=$?" >> gpurun_out/r2e/parity.log
timeout 900 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -k "c3" >> gpurun_out/r2e/parity.log 2>&1
echo "rc=$?" >> gpurun_out/r2e/parity.log
for k in 1 2; do
timeout 900 python tools/ab_time.py c3o12 8 "" >> gpurun_out/r2e/ab_c3o12.jsonl 2>&1
timeout 900 python tools/ab_time.py c3o16 8 "" >> gpurun_out/r2e/ab_c3o16.jsonl 2>&1
done
timeout 1200 python bench.py --config c4 --force-slabs --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2e/slab_c4.json 2> gpurun_out/r2e/slab_c4.err
echo "rc=$?" >> gpurun_out/r2e/slab_c4.err
tools/ncu_one.sh r2_vec_c4 c4 "acoustic3d_vec_kernel<.int.4, .bool.1, .int.8"
tools/ncu_one.sh r2_vec_c5fwd c5 "acoustic3d_vec_kernel<.int.4, .bool.1, .int.8"
tools/ncu_one.sh r2_vecgrad_c5 c5 "acoustic3d_vec_kernel<.int.4, .bool.0, .int.4, .bool.1" 5
tools/ncu_one.sh r2_vecq_c3o12b c3o12 "acoustic3d_vecq_kernel"
tools/ncu_one.sh r2_vecq_c3o16 c3o16 "acoustic3d_vecq_kernel"
