# Round-2 final-state validation after the a0-queue / last-warp-refills defaults:
# smoke, full GPU suite, bench lines for every config, ncu captures of the
# kernels whose default changed, C4 launch list.
set -u
bash tools/final_check.sh
bash tools/ncu_one.sh r2b_vecaq_c4 c4 "acoustic3d_vec_kernel<4, true, 16" 10
bash tools/ncu_one.sh r2b_vecq_last_c3o12 c3o12 "acoustic3d_vecq_kernel<6, true, 4, true>" 10
bash tools/ncu_one.sh r2b_vecq_c3o16 c3o16 "acoustic3d_vecq_kernel<8, true, 4" 10
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 200 --csv \
  --log-file gpurun_out/final/c4_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
