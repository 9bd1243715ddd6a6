# slab v2: slab parts (32-slice groups), launch bounds 3 CTAs/SM, unsigned variants
mkdir -p gpurun_out
for v in 15 115; do
WAMGPU_SLAB_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_parity3d.py -q -x > gpurun_out/p3d_v$v.log 2>&1; echo "parity3d v$v rc=$?"; tail -1 gpurun_out/p3d_v$v.log
done
for v in 9 12 15 16 17 18 19 115 118 109 112; do
WAMGPU_SLAB_VARIANT=$v timeout 600 python bench.py --config cfg5 --steps 1 --warmup 3 --iters 6 --no-cpu-baseline > gpurun_out/b5_v$v.json 2>gpurun_out/b5_v$v.err
tail -1 gpurun_out/b5_v$v.json | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('cfg5 v$v it/s',round(d['value'],2),'fwd',round(k['fwd_avg_ms'],3),'back',round(k['back_avg_ms'],3),d['clocks']['sm_mhz'])"
done
