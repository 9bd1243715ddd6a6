# banded 3D forward: parity on small stacks (forced bands), cfg4 band-size sweep, cfg4 expansion trace
python -m pytest tests/test_gpu_parity3d.py -x -q > gpurun_out/s5_pytest3d.log 2>&1; echo pytest rc=$?
tail -n 3 gpurun_out/s5_pytest3d.log
for mb in 0 48 24 96 12; do
  echo "== WAMGPU_FWD_BAND_MB=$mb"
  WAMGPU_FWD_BAND_MB=$mb python scripts/cfg4_iters.py cfg4 40 2>&1 | tail -n 2
done > gpurun_out/s5_band_sweep.log 2>&1
cat gpurun_out/s5_band_sweep.log
WAMGPU_TRACE_HOST=1 python scripts/time_expand.py cfg4 > gpurun_out/s5_expand_trace_cfg4.log 2>&1
tail -n 30 gpurun_out/s5_expand_trace_cfg4.log
