# slab v2 round 2: parity, variant times, ncu of variants 1/2/3
mkdir -p gpurun_out
for v in 0 3; do
WAMGPU_SLAB_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_parity3d.py -q -x > gpurun_out/p3d_v$v.log 2>&1; echo "parity3d v$v rc=$?"; tail -1 gpurun_out/p3d_v$v.log
done
for v in 3 8 9 10; do
WAMGPU_SLAB_VARIANT=$v timeout 600 python bench.py --config cfg5 --steps 1 --warmup 3 --iters 6 --no-cpu-baseline > gpurun_out/b5_v$v.json 2>gpurun_out/b5_v$v.err
tail -1 gpurun_out/b5_v$v.json | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('cfg5 v$v it/s',round(d['value'],2),'fwd',round(k['fwd_avg_ms'],3),'back',round(k['back_avg_ms'],3),d['clocks']['sm_mhz'])"
done
for v in 1 2 3; do
WAMGPU_SLAB_VARIANT=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_forward3|k_back3|k_fwd3s|k_back3s" -s 2 -c 2 -o gpurun_out/ncu3d_v$v python bench.py --config cfg5 --steps 1 --warmup 0 --iters 2 --no-cpu-baseline > gpurun_out/ncu3d_v$v.log 2>&1; echo "ncu v$v rc=$?"
done
