mkdir -p gpurun_out
for v in 0 1 2 3 4 0 1; do
WAMGPU_WALK_VARIANT=$v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/sw29_$v.log 2>&1
tail -1 gpurun_out/sw29_$v.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('wv',$v,round(d['value'],1),round(k['per_step_ms']['expand'],2))"
done
WAMGPU_WALK_VARIANT=4 timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
