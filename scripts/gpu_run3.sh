mkdir -p gpurun_out
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for fg in 1 2 4; do
WAMGPU_FG=$fg timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_fg$fg.log 2>&1; echo "bench fg=$fg rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/bench_cfg2_fg$fg.log').read().strip().splitlines()[-1]);print(d['value'],d['e2e']['value'],json.dumps(d['kernels']))"
done
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --iters 2"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_walk|k_forward|k_back" -c 3 -o gpurun_out/prof_cfg2 $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
