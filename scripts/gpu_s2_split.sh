# 3D split software pipeline (U rounds) at cfg3; slab part-launches at cfg4 AM
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity3d.py -q -x > gpurun_out/p3d_sp.log 2>&1; echo "parity3d rc=$?"; tail -1 gpurun_out/p3d_sp.log
for v in 0 3 4; do
WAMGPU_SPLIT_VARIANT=$v timeout 600 python bench.py --config cfg3 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/b3_sp$v.json 2>gpurun_out/b3_sp$v.err
tail -1 gpurun_out/b3_sp$v.json | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('cfg3 split v$v it/s',round(d['value'],2),k['per_step_ms'],d['clocks']['sm_mhz'])"
done
for v in 112 120 121; do
WAMGPU_SLAB_VARIANT=$v timeout 900 python bench.py --config cfg4 --algo am --iters 3 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/b4_v$v.json 2>gpurun_out/b4_v$v.err
tail -1 gpurun_out/b4_v$v.json | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('cfg4-am v$v it/s',round(d['value'],3),'fwd',round(k['fwd_avg_ms'],3),'back',round(k['back_avg_ms'],3),d['clocks']['sm_mhz'])"
done
