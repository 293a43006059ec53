set -u
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variant" > gpurun_out/ab/tests_variants.log 2>&1; tail -3 gpurun_out/ab/tests_variants.log
bash tools/ncu_one.sh r2b_vecaq_c4 c4 "acoustic3d_vec_kernel<.int.4, .bool.1, .int.16, .bool.0, .int.16, .int.1, .bool.1" 10
bash tools/ncu_one.sh r2b_vecq_last_c3o12 c3o12 "acoustic3d_vecq_kernel<.int.6, .bool.1, .int.4, .bool.1" 10
bash tools/ncu_one.sh r2b_vecq_c3o16 c3o16 "acoustic3d_vecq_kernel<.int.8, .bool.1, .int.4, .bool.0" 10
