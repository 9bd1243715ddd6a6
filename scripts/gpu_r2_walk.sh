# 3D walks with the tree bits in global memory (more CTAs per SM): parity, then expansion traces
mkdir -p gpurun_out/walk
timeout 900 python -m pytest tests/test_gpu_parity3d.py tests/test_gpu_sharded3d.py -x -q > gpurun_out/walk/pytest.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/walk/pytest.log
for cfg in cfg3 cfg4; do
WAMGPU_TRACE_HOST=1 timeout 900 python scripts/time_expand.py $cfg > gpurun_out/walk/trace_$cfg.log 2>&1; echo "$cfg rc=$?"
grep -E "expand at|Z walk|emit walk" gpurun_out/walk/trace_$cfg.log | tail -n 12
done
