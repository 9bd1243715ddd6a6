mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for fv in 0 1 2 3 4 5 6 7; do
WAMGPU_FWD_VARIANT=$fv WAMGPU_BACK_VARIANT=4 timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/sw_f$fv.log 2>&1
tail -1 gpurun_out/sw_f$fv.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('fwd',$fv,round(d['value'],1),round(k['fwd_avg_ms'],4),round(k['fwd_frac'],3),round(k['back_avg_ms'],4),round(k['per_step_ms']['expand'],1))"
done
for bv in 0 1 2 3 4; do
WAMGPU_BACK_VARIANT=$bv timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/sw_b$bv.log 2>&1
tail -1 gpurun_out/sw_b$bv.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('back',$bv,round(d['value'],1),round(k['back_avg_ms'],4),round(k['back_frac'],3))"
done
