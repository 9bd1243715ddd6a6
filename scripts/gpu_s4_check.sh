# Session-4 re-entry check at HEAD: smoke, full GPU tests, default bench (cfg2),
# 3D bench lines after the 3D Phi_A change (cfg3, cfg5, cfg4).
mkdir -p gpurun_out/s4
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/s4/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s4/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/s4/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s4/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/s4/r04_cfg2.json 2> gpurun_out/s4/r04_cfg2.err; echo "bench rc=$?"
for cfg in cfg3 cfg5; do
timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 > gpurun_out/s4/r04_$cfg.json 2> gpurun_out/s4/r04_$cfg.err; echo "$cfg rc=$?"
done
timeout 1500 python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s4/r04_cfg4.json 2> gpurun_out/s4/r04_cfg4.err; echo "cfg4 rc=$?"
