# Session-3 evidence: full GPU tests + smoke, default bench (cfg2 + CPU baseline),
# 3D bench lines after the slab register fix (cfg5, cfg3, cfg4), cfg4 shard at R=8.
mkdir -p gpurun_out/ev3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/ev3/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev3/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/ev3/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ev3/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ev3/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/ev3/r03_cfg2.json 2> gpurun_out/ev3/r03_cfg2.err; echo "bench rc=$?"
for cfg in cfg5 cfg3 cfg1; do
timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 > gpurun_out/ev3/r03_$cfg.json 2> gpurun_out/ev3/r03_$cfg.err; echo "$cfg rc=$?"
done
timeout 1500 python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ev3/r03_cfg4.json 2> gpurun_out/ev3/r03_cfg4.err; echo "cfg4 rc=$?"
timeout 1500 python bench.py --config cfg4 --shard 8 --view-groups 8 --steps 1 --warmup 3 > gpurun_out/ev3/r03_cfg4_R8_v8.json 2> gpurun_out/ev3/r03_cfg4_R8_v8.err; echo "cfg4 shard rc=$?"
