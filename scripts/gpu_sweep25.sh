mkdir -p gpurun_out
for v in 0 50 51 52 53 54 0; do
WAMGPU_FWD_VARIANT=$v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/sw25_$v.log 2>&1
tail -1 gpurun_out/sw25_$v.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('fv',$v,round(d['value'],1),round(k['fwd_avg_ms'],4),round(k['fwd_frac'],3),d['roofline']['frac'] if 'roofline' in d else '')"
done
WAMGPU_FWD_VARIANT=50 timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
