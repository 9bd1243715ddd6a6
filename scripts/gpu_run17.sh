mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for cfg in cfg2 cfg3; do
timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --config $cfg > gpurun_out/b_$cfg.log 2>&1
tail -1 gpurun_out/b_$cfg.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('$cfg',round(d['value'],2),k.get('per_step_ms'))"
done
