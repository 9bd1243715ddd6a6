# Round-2 session-4 baseline at HEAD: all GPU tests (incl. BASELINE-size fixtures cfg2/cfg3/cfg5),
# default bench (cfg4) + reference arm, cfg4 launch list.
mkdir -p gpurun_out/base
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/base/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/base/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/base/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/base/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/base/pytest_gpu.log
( time timeout 1200 python bench.py > gpurun_out/base/r06_cfg4.json 2> gpurun_out/base/r06_cfg4.err ) 2>&1 | tail -3; echo "bench rc=$?"
( time timeout 900 python bench.py --impl reference > gpurun_out/base/r06_cfg4_reference.json 2> gpurun_out/base/ref.err ) 2>&1 | tail -3; echo "ref rc=$?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/base/launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/base/ncu_ll.log 2>&1; echo "ncu-ll rc=$?"
python scripts/launches.py gpurun_out/base/launches_cfg4.csv > gpurun_out/base/launches_cfg4.txt; head -30 gpurun_out/base/launches_cfg4.txt
