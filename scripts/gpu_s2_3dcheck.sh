# new slab default (variant 112): full GPU tests, cfg5/cfg3/cfg4 bench lines
mkdir -p gpurun_out/bench
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for cfg in cfg5 cfg3; do
timeout 900 python bench.py --config $cfg --steps 2 --warmup 3 > gpurun_out/bench/r02_$cfg.json 2> gpurun_out/bench/r02_$cfg.err; echo "$cfg rc=$?"
tail -1 gpurun_out/bench/r02_$cfg.json | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('$cfg',round(d['value'],2),'e2e',round(d['e2e']['value'],2),'fwd',round(k['fwd_avg_ms'],3),'back',round(k['back_avg_ms'],3),k['per_step_ms'],d['clocks'],'cpu',d['cpu_baseline'] and d['cpu_baseline']['value'])"
done
timeout 1500 python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench/r02_cfg4.json 2> gpurun_out/bench/r02_cfg4.err; echo "cfg4 rc=$?"
tail -1 gpurun_out/bench/r02_cfg4.json | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('cfg4',round(d['value'],3),'e2e',round(d['e2e']['value'],3),'fwd',round(k['fwd_avg_ms'],3),'back',round(k['back_avg_ms'],3),k['per_step_ms'],d['clocks'])"
