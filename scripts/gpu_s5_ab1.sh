# A = Morton list build (old conversions, k_split3h_e); B = A + IMAD.WIDE conversions; C (in-tree) = B + k_split3p
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity3d.py tests/test_gpu_sharded3d.py tests/test_gpu_guards.py -m gpu -x -q > gpurun_out/s5_ab1_pytest.log 2>&1; tail -5 gpurun_out/s5_ab1_pytest.log
run() { # tag config env...
  tag=$1; cfg=$2; shift 2
  env "$@" timeout 1200 python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s5_ab1_${cfg}_$tag.log 2>&1
  tail -1 gpurun_out/s5_ab1_${cfg}_$tag.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('$cfg $tag',round(d['value'],3),{a:round(b,1) for a,b in k['per_step_ms'].items()},d['clocks']['sm_mhz'])"
}
A=$PWD/paper_1508_04458_b200/_build/libwamgpu_A.so
B=$PWD/paper_1508_04458_b200/_build/libwamgpu_B.so
for cfg in cfg4 cfg3; do
run A_rowmajor $cfg WAMGPU_LIB=$A WAMGPU_SPLIT_ORDER=0
run A_morton $cfg WAMGPU_LIB=$A
run B_imad $cfg WAMGPU_LIB=$B
run C_split3p $cfg X=1
run C_split3p_notrick $cfg WAMGPU_SPLIT_VARIANT=8
run C_oldsplit $cfg WAMGPU_SPLIT_VARIANT=6
run C_split3p_rowmajor $cfg WAMGPU_SPLIT_ORDER=0
done
run B_imad cfg5 WAMGPU_LIB=$B
run A cfg5 WAMGPU_LIB=$A
