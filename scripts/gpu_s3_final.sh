# Session-3 final evidence for the default bench (cfg2): bench line with CPU
# baseline, reference arm, ncu launch list of the same command, smoke + GPU tests.
mkdir -p gpurun_out/fin
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/fin/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fin/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/fin/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/fin/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/fin/r03_cfg2.json 2> gpurun_out/fin/r03_cfg2.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/fin/r03_cfg2_reference.json 2> gpurun_out/fin/ref.err; echo "ref rc=$?"
timeout 900 python bench.py --config cfg1 --steps 3 --warmup 3 > gpurun_out/fin/r03_cfg1.json 2> gpurun_out/fin/r03_cfg1.err; echo "cfg1 rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/fin/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/fin/ncu_ll.log 2>&1; echo "ncu-ll rc=$?"
python scripts/launches.py gpurun_out/fin/launches_cfg2.csv > gpurun_out/fin/launches_cfg2.txt; head -16 gpurun_out/fin/launches_cfg2.txt
timeout 900 ncu --set full --clock-control none -f --import-source on -k regex:"k_phiA_fwd|k_phiA_back" -s 4 -c 2 -o gpurun_out/fin/ncu_phi python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/fin/ncu_phi.log 2>&1; echo "ncu-phi rc=$?"
