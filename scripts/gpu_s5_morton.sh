# Morton-ordered split list (WAMGPU_SPLIT_ORDER=1, default) against row-major (0); z-activity statistics
mkdir -p gpurun_out
for c in cfg4 cfg3; do for o in 0 1 0 1; do
WAMGPU_SPLIT_ORDER=$o timeout 1200 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s5_mo_${c}_$o.log 2>&1
tail -1 gpurun_out/s5_mo_${c}_$o.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('$c order',$o,round(d['value'],3),{a:round(b,1) for a,b in k['per_step_ms'].items()},d['clocks']['sm_mhz'])"
done; done
timeout 900 python scripts/tree_zstats.py cfg4 > gpurun_out/s5_zstats_cfg4.log 2>&1; cat gpurun_out/s5_zstats_cfg4.log
timeout 900 python scripts/tree_zstats.py cfg3 > gpurun_out/s5_zstats_cfg3.log 2>&1; cat gpurun_out/s5_zstats_cfg3.log
