# evidence at HEAD (double-operand coarse back projection in): full GPU suite, smoke, contract line, other configs
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -x -q > gpurun_out/s5_final4_pytest.log 2>&1; tail -3 gpurun_out/s5_final4_pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/s5_final4_smoke.log 2>&1; tail -1 gpurun_out/s5_final4_smoke.log
timeout 1800 python bench.py > gpurun_out/s5_final4_cfg4.log 2>&1; tail -1 gpurun_out/s5_final4_cfg4.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('cfg4',round(d['value'],3),round(d['e2e']['value'],3),{a:round(b,1) for a,b in k['per_step_ms'].items()},d['clocks'],d.get('device_memory_gib'),d['cpu_baseline']['value'],d['gpu_launches'])"
for c in cfg3 cfg2 cfg1 cfg5; do
timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s5_final4_$c.log 2>&1; tail -1 gpurun_out/s5_final4_$c.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('$c',round(d['value'],3),round(d['e2e']['value'],3),{a:round(b,1) for a,b in k['per_step_ms'].items()},d.get('device_memory_gib'),d['gpu_launches'])"
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/s5_launches4_cfg4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s5_ncu_launches4.log 2>&1; echo "launch list rc=$?"
gzip -f gpurun_out/s5_launches4_cfg4.csv
