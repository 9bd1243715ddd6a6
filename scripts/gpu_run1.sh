mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -5 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config cfg1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg1.log 2>&1; echo "bench1 rc=$?"
tail -3 gpurun_out/bench_cfg1.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_cfg2.log 2>&1; echo "bench2 rc=$?"
tail -3 gpurun_out/bench_cfg2.log
