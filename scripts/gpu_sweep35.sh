mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity3d.py -x -q 2>&1 | tail -2; echo parity-done
for v in 0 1 0; do
WAMGPU_SPLIT_VARIANT=$v timeout 600 python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/sw35_$v.log 2>&1
tail -1 gpurun_out/sw35_$v.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('sv',$v,round(d['value'],2),{a:round(b,1) for a,b in k['per_step_ms'].items()})"
done
