mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for t in 0 1; do
WAMGPU_MU_TILED=$t timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/sw_t$t.log 2>&1
tail -1 gpurun_out/sw_t$t.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('tiled',$t,round(d['value'],1),round(k['fwd_avg_ms'],4),round(k['fwd_frac'],3),round(k['back_avg_ms'],4),round(k['per_step_ms']['expand'],1))"
done
