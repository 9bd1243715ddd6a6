# Session-4 evidence for the default bench (cfg2) after the counting placement:
# smoke, GPU tests, bench line with CPU baseline, reference arm, cfg1, ncu --set
# full of the dominant kernels (k_fwd_patch, k_back) and the expansion kernels.
mkdir -p gpurun_out/fin4
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/fin4/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin4/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fin4/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/fin4/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/fin4/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/fin4/r04_cfg2.json 2> gpurun_out/fin4/r04_cfg2.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/fin4/r04_cfg2_reference.json 2> gpurun_out/fin4/ref.err; echo "ref rc=$?"
timeout 900 python bench.py --config cfg1 --steps 3 --warmup 3 > gpurun_out/fin4/r04_cfg1.json 2> gpurun_out/fin4/r04_cfg1.err; echo "cfg1 rc=$?"
timeout 900 ncu --set full --clock-control none -f --import-source on -k regex:"k_fwd_patch|k_back<|k_key_place|k_key_hist|k_walk_lv" -s 20 -c 8 -o gpurun_out/fin4/ncu_cfg2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/fin4/ncu_cfg2.log 2>&1; echo "ncu rc=$?"
