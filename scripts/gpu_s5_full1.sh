# full GPU suite with coarse projections (2D and 3D) and k_split3c v11 as defaults; all five configs
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -x -q > gpurun_out/s5_full1_pytest.log 2>&1; tail -5 gpurun_out/s5_full1_pytest.log
run() { # tag config env...
  tag=$1; cfg=$2; shift 2
  env "$@" timeout 1200 python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s5_full1_${cfg}_$tag.log 2>&1
  tail -1 gpurun_out/s5_full1_${cfg}_$tag.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('$cfg $tag',round(d['value'],3),round(d['e2e']['value'],3),{a:round(b,1) for a,b in k['per_step_ms'].items()},d['clocks']['sm_mhz'], d['final_objective'], [e.get('tree_sha256','')[:8] for e in (d.get('parity') or {}).get('expansions',[])], 'upd/s %.3e' % d['ray_voxel_updates_per_s'])" || tail -5 gpurun_out/s5_full1_${cfg}_$tag.log
}
run coarse cfg2 X=1
run fine cfg2 WAMGPU_COARSE=0
run coarse cfg1 X=1
run fine cfg1 WAMGPU_COARSE=0
run coarse cfg4 X=1
run coarse cfg3 X=1
run am cfg5 X=1
