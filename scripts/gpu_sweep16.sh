mkdir -p gpurun_out
for t in 1 0; do for fv in 4 7 3 8 1; do
WAMGPU_MU_TILED=$t WAMGPU_FWD_VARIANT=$fv timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/sw.log 2>&1
tail -1 gpurun_out/sw.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('tiled',$t,'fv',$fv,round(d['value'],1),round(k['fwd_avg_ms'],4),round(k['fwd_frac'],3))"
done; done
