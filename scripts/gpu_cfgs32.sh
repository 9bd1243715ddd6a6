mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
for cfg in cfg1 cfg5 cfg3; do
timeout 900 python bench.py --config $cfg --steps 2 --warmup 3 > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err; echo "$cfg rc=$?"
tail -1 gpurun_out/bench_$cfg.json | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('$cfg',round(d['value'],2),'e2e',round(d['e2e']['value'],2),'roof',round(d['roofline']['frac'],3),'gather',k.get('gather_gbs'),k['per_step_ms'],'cpu',d['cpu_baseline'] and d['cpu_baseline']['value'])"
done
timeout 1500 python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4 rc=$?"
tail -1 gpurun_out/bench_cfg4.json | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('cfg4',round(d['value'],3),'e2e',round(d['e2e']['value'],3),'roof',round(d['roofline']['frac'],3),k['per_step_ms'],d['clocks'])"
