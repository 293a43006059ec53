# Stress: the whole GPU suite with sf_plan_invoke's overlapped form forced at
# every size (32-plane chunks), so every 3D acoustic parity case with more than
# 32 planes also runs through the time-skewed upload / copy back.
set -u
mkdir -p gpurun_out/stress
SF_IO_OVERLAP=1 SF_IO_CHUNK_PLANES=32 timeout 2400 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_configs.py::test_c4_full_time_loop_vs_reference > gpurun_out/stress/forced_overlap_suite.log 2>&1
echo "rc=$?" >> gpurun_out/stress/forced_overlap_suite.log
tail -4 gpurun_out/stress/forced_overlap_suite.log
