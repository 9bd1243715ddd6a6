mkdir -p gpurun_out
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for cfg in cfg1 cfg2; do
timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$cfg.log 2>&1; echo "bench $cfg rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_$cfg.log').read().strip().splitlines()[-1]);print(d['value'],d['e2e']['value'],json.dumps(d['kernels']), json.dumps(d['tree']))"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
python scripts/launches.py gpurun_out/launches_cfg2.csv > gpurun_out/launches_cfg2.txt; head -14 gpurun_out/launches_cfg2.txt
