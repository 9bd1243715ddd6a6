mkdir -p gpurun_out
for v in 3 4 5 6 7 3; do
WAMGPU_SPLIT_VARIANT=$v timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/sw27_$v.log 2>&1
tail -1 gpurun_out/sw27_$v.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('sv',$v,round(d['value'],1),k['per_step_ms'])"
done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
