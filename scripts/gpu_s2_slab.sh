# slab SpMM v2: parity under each variant, then per-variant forward/back times at cfg5 (AM) and cfg3 (WAM)
mkdir -p gpurun_out
for v in 0 2 3; do
WAMGPU_SLAB_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_parity3d.py -q -x > gpurun_out/p3d_v$v.log 2>&1; echo "parity3d v$v rc=$?"; tail -1 gpurun_out/p3d_v$v.log
done
for v in 1 0 2 3 4 5 6 7; do
WAMGPU_SLAB_VARIANT=$v timeout 600 python bench.py --config cfg5 --steps 1 --warmup 3 --iters 6 --no-cpu-baseline > gpurun_out/b5_v$v.json 2>gpurun_out/b5_v$v.err
tail -1 gpurun_out/b5_v$v.json | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('cfg5 v$v it/s',round(d['value'],2),'fwd',round(k['fwd_avg_ms'],3),'back',round(k['back_avg_ms'],3),d['clocks']['sm_mhz'])"
done
for v in 1 0 2; do
WAMGPU_SLAB_VARIANT=$v timeout 600 python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/b3_v$v.json 2>gpurun_out/b3_v$v.err
tail -1 gpurun_out/b3_v$v.json | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('cfg3 v$v it/s',round(d['value'],2),'fwd',round(k['fwd_avg_ms'],3),'back',round(k['back_avg_ms'],3),k['per_step_ms'],d['clocks']['sm_mhz'])"
done
