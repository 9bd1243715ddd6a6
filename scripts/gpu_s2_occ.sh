# occupancy variants: slab SpMM (U=2 / 4-warp CTAs) at cfg5, 3D split E=2 (80 registers) at cfg3
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity3d.py -q -x > gpurun_out/p3d_occ.log 2>&1; echo "parity3d rc=$?"; tail -1 gpurun_out/p3d_occ.log
for v in 112 113 114 115 116; do
WAMGPU_SLAB_VARIANT=$v timeout 600 python bench.py --config cfg5 --steps 1 --warmup 3 --iters 6 --no-cpu-baseline > gpurun_out/b5_o$v.json 2>gpurun_out/b5_o$v.err
tail -1 gpurun_out/b5_o$v.json | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('cfg5 v$v it/s',round(d['value'],2),'fwd',round(k['fwd_avg_ms'],3),'back',round(k['back_avg_ms'],3),d['clocks']['sm_mhz'])"
done
for v in 0 5; do
WAMGPU_SPLIT_VARIANT=$v timeout 600 python bench.py --config cfg3 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/b3_sp$v.json 2>gpurun_out/b3_sp$v.err
tail -1 gpurun_out/b3_sp$v.json | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('cfg3 split v$v it/s',round(d['value'],2),{a:round(b,1) for a,b in k['per_step_ms'].items()},d['clocks']['sm_mhz'])"
done
