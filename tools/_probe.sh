mkdir -p gpurun_out/probe
(lscpu; free -g; nproc; nvidia-smi; df -h /tmp .) > gpurun_out/probe/machine.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/probe/gputest.log 2>&1
echo rc=$? >> gpurun_out/probe/gputest.log
