# k_split3c (cp.async ring, CTA per block) variants against k_split3p (0) and k_split3h_e (6); Morton list, shift conversions
mkdir -p gpurun_out
for v in 10 11; do
WAMGPU_SPLIT_VARIANT=$v timeout 900 python -m pytest tests/test_gpu_parity3d.py tests/test_gpu_sharded3d.py -m gpu -x -q > gpurun_out/s5_ab2_pytest_$v.log 2>&1; tail -3 gpurun_out/s5_ab2_pytest_$v.log
done
run() { # tag config env...
  tag=$1; cfg=$2; shift 2
  env "$@" timeout 1200 python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s5_ab2_${cfg}_$tag.log 2>&1
  tail -1 gpurun_out/s5_ab2_${cfg}_$tag.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('$cfg $tag',round(d['value'],3),{a:round(b,1) for a,b in k['per_step_ms'].items()},d['clocks']['sm_mhz'], d['final_objective'])"
}
for cfg in cfg4 cfg3; do
for v in 0 6 10 11 12 13 14; do run v$v $cfg WAMGPU_SPLIT_VARIANT=$v; done
run v10_rowmajor $cfg WAMGPU_SPLIT_VARIANT=10 WAMGPU_SPLIT_ORDER=0
done
