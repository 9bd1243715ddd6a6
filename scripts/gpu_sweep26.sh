mkdir -p gpurun_out
for v in 0 10 11 12 13 14 15; do
WAMGPU_BACK_VARIANT=$v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/sw26_$v.log 2>&1
tail -1 gpurun_out/sw26_$v.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('bv',$v,round(d['value'],1),'fwd',round(k['fwd_avg_ms'],4),'back',round(k['back_avg_ms'],4),round(k['back_frac'],3))"
done
WAMGPU_BACK_VARIANT=10 timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
