# Host-traced expansion phases of the cfg3 R=8 detached shard (views only).
mkdir -p gpurun_out/s4t
WAMGPU_TRACE_HOST=1 timeout 600 python bench.py --config cfg3 --shard 8 --view-groups 8 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/s4t/shard8.json 2> gpurun_out/s4t/shard8_trace.log; echo "rc=$?"
grep -i "expand" gpurun_out/s4t/shard8_trace.log | tail -40
