mkdir -p gpurun_out
for v in 0 2 1; do
WAMGPU_SPLIT_VARIANT=$v timeout 1200 python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/sw36_$v.log 2>&1
tail -1 gpurun_out/sw36_$v.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('sv',$v,round(d['value'],3),{a:round(b,1) for a,b in k['per_step_ms'].items()},d['clocks']['sm_mhz'])"
done
