# Session-5 baseline at HEAD: GPU tests, smoke, cfg4/cfg3/cfg2 bench lines.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/s5_pytest_gpu.log 2>&1; tail -3 gpurun_out/s5_pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/s5_smoke.log 2>&1; tail -1 gpurun_out/s5_smoke.log
for c in cfg4 cfg3 cfg2; do
timeout 1500 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s5_$c.log 2>&1
tail -1 gpurun_out/s5_$c.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('$c',round(d['value'],3),round(d['e2e']['value'],3),{a:round(b,1) for a,b in k['per_step_ms'].items()},d['clocks']['sm_mhz'])"
done
