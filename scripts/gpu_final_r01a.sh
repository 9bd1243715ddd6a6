# Round-1 evidence refresh: tests, default bench (+CPU baseline), reference arm,
# ncu launch list of the same bench command, DRAM bytes of the dominant kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_cfg2.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_cfg2.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_ref_cfg2.json | head -c 800
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_ll.log 2>&1; echo "ncu-ll rc=$?"
python scripts/launches.py gpurun_out/launches_cfg2.csv > gpurun_out/launches_cfg2.txt; head -16 gpurun_out/launches_cfg2.txt
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:"k_fwd_patch|k_back<|k_split|k_walk_lv" -s 20 -c 8 --csv --log-file gpurun_out/dram_cfg2.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_dram.log 2>&1; echo "ncu-dram rc=$?"
