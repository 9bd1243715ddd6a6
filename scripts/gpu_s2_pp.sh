# ping-pong slab kernel (no register copies, 128-register cap): parity + cfg5/cfg4 per-pass times
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity3d.py -q -x > gpurun_out/p3d_pp.log 2>&1; echo "parity3d rc=$?"; tail -1 gpurun_out/p3d_pp.log
for v in 112 109 103; do
WAMGPU_SLAB_VARIANT=$v timeout 600 python bench.py --config cfg5 --steps 1 --warmup 3 --iters 6 --no-cpu-baseline > gpurun_out/b5_pp$v.json 2>gpurun_out/b5_pp$v.err
tail -1 gpurun_out/b5_pp$v.json | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('cfg5 pp v$v it/s',round(d['value'],2),'fwd',round(k['fwd_avg_ms'],3),'back',round(k['back_avg_ms'],3),d['clocks']['sm_mhz'])"
done
timeout 900 python bench.py --config cfg4 --algo am --iters 3 --steps 1 --warmup 2 --no-cpu-baseline > gpurun_out/b4_pp.json 2>gpurun_out/b4_pp.err
tail -1 gpurun_out/b4_pp.json | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('cfg4-am pp it/s',round(d['value'],3),'fwd',round(k['fwd_avg_ms'],3),'back',round(k['back_avg_ms'],3),d['clocks']['sm_mhz'])"
