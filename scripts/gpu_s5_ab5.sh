# k_split3c with sector-friendly chunk mapping (each cp.async instruction covers whole 32-byte sectors)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_coarse.py tests/test_gpu_parity3d.py tests/test_gpu_sharded3d.py tests/test_gpu_guards.py -m gpu -x -q > gpurun_out/s5_ab5_pytest.log 2>&1; tail -5 gpurun_out/s5_ab5_pytest.log
run() { # tag config env...
  tag=$1; cfg=$2; shift 2
  env "$@" timeout 1200 python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s5_ab5_${cfg}_$tag.log 2>&1
  tail -1 gpurun_out/s5_ab5_${cfg}_$tag.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('$cfg $tag',round(d['value'],3),{a:round(b,1) for a,b in k['per_step_ms'].items()},d['clocks']['sm_mhz'], d['final_objective'], [e.get('tree_sha256','')[:8] for e in d['parity']['expansions']], 'upd/s %.3e' % d['ray_voxel_updates_per_s'])" || tail -5 gpurun_out/s5_ab5_${cfg}_$tag.log
}
for cfg in cfg4 cfg3; do
run v12 $cfg X=1
run v10 $cfg WAMGPU_SPLIT_VARIANT=10
run v11 $cfg WAMGPU_SPLIT_VARIANT=11
run v13 $cfg WAMGPU_SPLIT_VARIANT=13
done
