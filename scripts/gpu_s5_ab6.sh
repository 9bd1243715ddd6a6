# k_split3c with per-entry multipliers precomputed at batch staging (8 fp64 per entry in shared memory)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_coarse.py tests/test_gpu_parity3d.py tests/test_gpu_sharded3d.py tests/test_gpu_guards.py -m gpu -x -q > gpurun_out/s5_ab6_pytest.log 2>&1; tail -3 gpurun_out/s5_ab6_pytest.log
run() { # tag config env...
  tag=$1; cfg=$2; shift 2
  env "$@" timeout 1200 python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s5_ab6_${cfg}_$tag.log 2>&1
  tail -1 gpurun_out/s5_ab6_${cfg}_$tag.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('$cfg $tag',round(d['value'],3),round(d['e2e']['value'],3),{a:round(b,1) for a,b in k['per_step_ms'].items()},d['clocks']['sm_mhz'], d['final_objective'], [e.get('tree_sha256','')[:8] for e in (d.get('parity') or {}).get('expansions',[])], d.get('device_memory_gib'))" || tail -5 gpurun_out/s5_ab6_${cfg}_$tag.log
}
run v11 cfg4 X=1
run v10 cfg4 WAMGPU_SPLIT_VARIANT=10
run v11 cfg3 X=1
run v10 cfg3 WAMGPU_SPLIT_VARIANT=10
