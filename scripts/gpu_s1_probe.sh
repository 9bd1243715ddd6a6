set -x
nproc; free -g; lscpu | head -20; nvidia-smi -L
python -m pytest tests -m gpu -x -q > gpurun_out/s1_pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/s1_pytest_gpu.log
