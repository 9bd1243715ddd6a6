# small slab strides (P = 8/16/32 shards): parity; per-shard times at nz = 64/R (R = 1, 2, 4, 8) for cfg5 and cfg3
mkdir -p gpurun_out/shard
timeout 900 python -m pytest tests/test_gpu_parity3d.py -q -x > gpurun_out/p3d_smallp.log 2>&1; echo "parity3d rc=$?"; tail -3 gpurun_out/p3d_smallp.log
for cfg in cfg5 cfg3; do for nz in 64 32 16 8; do
timeout 900 python bench.py --config $cfg --nz $nz --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/shard/${cfg}_nz$nz.json 2>gpurun_out/shard/${cfg}_nz$nz.err
tail -1 gpurun_out/shard/${cfg}_nz$nz.json | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('$cfg nz=$nz it/s',round(d['value'],2),'ms/run',round(d['ms_per_step'],1),'fwd',round(k['fwd_avg_ms'],3),'back',round(k['back_avg_ms'],3),{a:round(b,1) for a,b in k['per_step_ms'].items()},d['clocks']['sm_mhz'])"
done; done
