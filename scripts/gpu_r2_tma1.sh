# on-the-fly TMA forward: parity on the small stacks, then cfg5 / cfg3 / cfg4 A/B (WAMGPU_FWD3T=0/1)
mkdir -p gpurun_out/tma1
timeout 600 python -m pytest tests/test_gpu_parity3d.py -x -q -k "on_the_fly" > gpurun_out/tma1/pytest.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -n 25 gpurun_out/tma1/pytest.log
[ $rc -ne 0 ] && exit 0
for cfg in cfg5 cfg3; do for t in 0 1; do
  echo "== $cfg WAMGPU_FWD3T=$t"; WAMGPU_FWD3T=$t timeout 600 python scripts/cfg4_iters.py $cfg 30 2>&1 | tail -n 2
done; done > gpurun_out/tma1/ab_cfg35.log 2>&1
cat gpurun_out/tma1/ab_cfg35.log
for t in 0 1; do
  echo "== cfg4 WAMGPU_FWD3T=$t"; WAMGPU_FWD3T=$t timeout 900 python scripts/cfg4_iters.py cfg4 20 2>&1 | tail -n 2
done > gpurun_out/tma1/ab_cfg4.log 2>&1
cat gpurun_out/tma1/ab_cfg4.log
