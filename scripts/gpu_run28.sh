mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
WAMGPU_TRACE_HOST=1 python scripts/time_expand.py cfg2 2>&1 | grep -E "walk|sort|^expand" | tail -12
timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --config cfg2 > gpurun_out/b_cfg2.log 2>&1
tail -1 gpurun_out/b_cfg2.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('cfg2',round(d['value'],2),k.get('per_step_ms'))"
