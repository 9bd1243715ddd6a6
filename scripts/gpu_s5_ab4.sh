# z-coarse projections (WAMGPU_COARSE=2, default) against in-plane only (1); default split = k_split3c v12; ncu of the split at the cfg4 final tree
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_coarse.py tests/test_gpu_parity3d.py tests/test_gpu_sharded3d.py tests/test_gpu_guards.py -m gpu -x -q > gpurun_out/s5_ab4_pytest.log 2>&1; tail -5 gpurun_out/s5_ab4_pytest.log
run() { # tag config env...
  tag=$1; cfg=$2; shift 2
  env "$@" timeout 1200 python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s5_ab4_${cfg}_$tag.log 2>&1
  tail -1 gpurun_out/s5_ab4_${cfg}_$tag.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('$cfg $tag',round(d['value'],3),{a:round(b,1) for a,b in k['per_step_ms'].items()},d['clocks']['sm_mhz'], d['final_objective'], [e.get('tree_sha256','')[:8] for e in d['parity']['expansions']], 'upd/s %.3e' % d['ray_voxel_updates_per_s'])" || tail -5 gpurun_out/s5_ab4_${cfg}_$tag.log
}
for cfg in cfg4 cfg3; do
run z $cfg X=1
run inplane $cfg WAMGPU_COARSE=1
done
python scripts/cfg4_iters.py cfg4 36 > gpurun_out/s5_ab4_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -f --import-source on -k regex:"k_split3c" -s 26 -c 1 -o /tmp/split4 python scripts/cfg4_iters.py cfg4 36 > gpurun_out/s5_ab4_ncu_split.log 2>&1; echo "ncu split rc=$?"
ncu -i /tmp/split4.ncu-rep --page raw --csv > gpurun_out/s5_split3c_raw.csv
ncu -i /tmp/split4.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/s5_split3c_src.csv.gz
ls -la gpurun_out | tail -5
