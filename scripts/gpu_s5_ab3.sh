# coarse projections (kernels3c.cuh) + k_split3c with dynamic scheduling and IMAD.WIDE conversions
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_coarse.py tests/test_gpu_parity3d.py tests/test_gpu_sharded3d.py tests/test_gpu_guards.py -m gpu -x -q > gpurun_out/s5_ab3_pytest.log 2>&1; tail -5 gpurun_out/s5_ab3_pytest.log
WAMGPU_SPLIT_VARIANT=10 timeout 900 python -m pytest tests/test_gpu_parity3d.py -m gpu -x -q > gpurun_out/s5_ab3_pytest_v10.log 2>&1; tail -3 gpurun_out/s5_ab3_pytest_v10.log
WAMGPU_SPLIT_VARIANT=11 timeout 900 python -m pytest tests/test_gpu_parity3d.py -m gpu -x -q > gpurun_out/s5_ab3_pytest_v11.log 2>&1; tail -3 gpurun_out/s5_ab3_pytest_v11.log
run() { # tag config env...
  tag=$1; cfg=$2; shift 2
  env "$@" timeout 1200 python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s5_ab3_${cfg}_$tag.log 2>&1
  tail -1 gpurun_out/s5_ab3_${cfg}_$tag.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('$cfg $tag',round(d['value'],3),{a:round(b,1) for a,b in k['per_step_ms'].items()},d['clocks']['sm_mhz'], d['final_objective'], [e.get('tree_sha256','')[:8] for e in d['parity']['expansions']])" || tail -5 gpurun_out/s5_ab3_${cfg}_$tag.log
}
for cfg in cfg4 cfg3; do
run fine_v6 $cfg WAMGPU_COARSE=0 WAMGPU_SPLIT_VARIANT=6
run coarse_v10 $cfg WAMGPU_SPLIT_VARIANT=10
run coarse_v11 $cfg WAMGPU_SPLIT_VARIANT=11
run coarse_v12 $cfg WAMGPU_SPLIT_VARIANT=12
run coarse_v13 $cfg WAMGPU_SPLIT_VARIANT=13
done
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
