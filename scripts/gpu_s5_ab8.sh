# z-coarse back projection over fp64 z-group sums (k_back3s XD, WAMGPU_COARSE_DBL=1 default) against fp32 hi/lo pairs (0)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_coarse.py tests/test_gpu_parity3d.py tests/test_gpu_sharded3d.py tests/test_gpu_guards.py tests/test_gpu_parity_big.py -m gpu -x -q > gpurun_out/s5_ab8_pytest.log 2>&1; tail -15 gpurun_out/s5_ab8_pytest.log
run() { # tag config env...
  tag=$1; cfg=$2; shift 2
  env "$@" timeout 1200 python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s5_ab8_${cfg}_$tag.log 2>&1
  tail -1 gpurun_out/s5_ab8_${cfg}_$tag.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('$cfg $tag',round(d['value'],3),round(d['e2e']['value'],3),{a:round(b,1) for a,b in k['per_step_ms'].items()},d['clocks']['sm_mhz'], d['final_objective'], [e.get('tree_sha256','')[:8] for e in (d.get('parity') or {}).get('expansions',[])])" || tail -5 gpurun_out/s5_ab8_${cfg}_$tag.log
}
run dbl cfg4 X=1
run hilo cfg4 WAMGPU_COARSE_DBL=0
run dbl cfg3 X=1
run hilo cfg3 WAMGPU_COARSE_DBL=0
