# Host-traced phases of each 2D wam_expand at cfg2.
mkdir -p gpurun_out/s4t2
WAMGPU_TRACE_HOST=1 timeout 600 python scripts/time_expand.py cfg2 > gpurun_out/s4t2/trace_cfg2.log 2>&1; echo "rc=$?"
grep -v "iter" gpurun_out/s4t2/trace_cfg2.log | tail -45
