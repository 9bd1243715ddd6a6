# full GPU suite again (coarse also under view shards without split update); root-only phase over the coarse path (WAMGPU_COARSE_ROOT=1) A/B
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -x -q > gpurun_out/s5_full2_pytest.log 2>&1; tail -5 gpurun_out/s5_full2_pytest.log
WAMGPU_COARSE_ROOT=1 timeout 900 python -m pytest tests/test_gpu_parity3d.py tests/test_gpu_coarse.py -m gpu -x -q > gpurun_out/s5_full2_pytest_root.log 2>&1; tail -3 gpurun_out/s5_full2_pytest_root.log
run() { # tag config env...
  tag=$1; cfg=$2; shift 2
  env "$@" timeout 1200 python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s5_full2_${cfg}_$tag.log 2>&1
  tail -1 gpurun_out/s5_full2_${cfg}_$tag.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('$cfg $tag',round(d['value'],3),round(d['e2e']['value'],3),{a:round(b,1) for a,b in k['per_step_ms'].items()},d['clocks']['sm_mhz'], d['final_objective'], [e.get('tree_sha256','')[:8] for e in (d.get('parity') or {}).get('expansions',[])], 'upd/s %.3e' % d['ray_voxel_updates_per_s'])" || tail -5 gpurun_out/s5_full2_${cfg}_$tag.log
}
run root cfg4 WAMGPU_COARSE_ROOT=1
run phiA cfg4 X=1
run root cfg3 WAMGPU_COARSE_ROOT=1
run phiA cfg3 X=1
