mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --config cfg3 --steps 2 --warmup 1 --cpu-iters 1 > gpurun_out/bench_cfg3.log 2>&1; echo "bench cfg3 rc=$?"
tail -1 gpurun_out/bench_cfg3.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['e2e']['value'],d['ray_voxel_updates_per_s'],json.dumps(d['kernels']['per_step_ms']),json.dumps(d['tree']),json.dumps(d['cpu_baseline']))"
timeout 2400 python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_cfg4.log 2>&1; echo "bench cfg4 rc=$?"
tail -1 gpurun_out/bench_cfg4.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['e2e']['value'],d['ray_voxel_updates_per_s'],json.dumps(d['kernels']['per_step_ms']),json.dumps(d['tree']))"
