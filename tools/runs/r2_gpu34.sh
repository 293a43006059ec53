# Full-time-loop parity of every config on the final kernels (a0 queue, last-
# warp-refills, residual-guarded reciprocal) and through sf_plan_invoke's
# overlapped upload / copy back: C1 500, C2 625, C3 order 8 500, C4 1000 steps
# bitwise vs the live reference; C5 at nt = 100 vs the port.
set -u
mkdir -p gpurun_out/long
SF_LONG_TESTS=1 timeout 3400 python -m pytest tests/test_gpu_configs.py -m gpu -x -v > gpurun_out/long/full_time_loop_parity.log 2>&1
echo "rc=$?" >> gpurun_out/long/full_time_loop_parity.log
tail -15 gpurun_out/long/full_time_loop_parity.log
