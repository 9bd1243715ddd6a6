mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_fused_ar.py -x -q > gpurun_out/pytest_ar.log 2>&1; echo "ar rc=$?"; tail -5 gpurun_out/pytest_ar.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b_cfg2.log 2>&1
tail -1 gpurun_out/b_cfg2.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('cfg2',round(d['value'],2),k.get('per_step_ms'))"
