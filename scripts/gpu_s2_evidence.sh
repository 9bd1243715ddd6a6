# Session-2 evidence refresh: tests + smoke, default bench (cfg2, with CPU baseline), reference arm,
# other configs, ncu launch list of the default bench command, DRAM bytes of the dominant kernels,
# ncu --set full of the top kernel (k_fwd_patch) and of the 3D slab forward at cfg5.
mkdir -p gpurun_out/ev
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/ev/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/ev/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/ev/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ev/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/ev/r02_cfg2.json 2> gpurun_out/ev/r02_cfg2.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/ev/r02_cfg2_reference.json 2> gpurun_out/ev/ref.err; echo "ref rc=$?"
for cfg in cfg1 cfg5 cfg3; do
timeout 900 python bench.py --config $cfg --steps 2 --warmup 3 > gpurun_out/ev/r02_$cfg.json 2> gpurun_out/ev/r02_$cfg.err; echo "$cfg rc=$?"
done
timeout 1500 python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ev/r02_cfg4.json 2> gpurun_out/ev/r02_cfg4.err; echo "cfg4 rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/ev/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ev/ncu_ll.log 2>&1; echo "ncu-ll rc=$?"
python scripts/launches.py gpurun_out/ev/launches_cfg2.csv > gpurun_out/ev/launches_cfg2.txt; head -12 gpurun_out/ev/launches_cfg2.txt
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_fwd_patch|k_back<|k_split<|k_walk_lv" -s 20 -c 8 --csv --log-file gpurun_out/ev/dram_cfg2.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ev/ncu_dram.log 2>&1; echo "ncu-dram rc=$?"
timeout 900 ncu --set full --clock-control none -f --import-source on -k regex:"k_fwd_patch|k_back<" -s 10 -c 2 -o /tmp/ncu_top python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ev/ncu_top.log 2>&1; echo "ncu-top rc=$?"
ncu -i /tmp/ncu_top.ncu-rep --page raw --csv > gpurun_out/ev/ncu_top_raw.csv
