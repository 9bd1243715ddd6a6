mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for cfg in cfg5 cfg3; do
timeout 1200 python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_$cfg.log 2>&1; echo "bench $cfg rc=$?"
tail -1 gpurun_out/bench_$cfg.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['e2e']['value'],d['ray_voxel_updates_per_s'],json.dumps(d['kernels']), json.dumps(d.get('tree')))"
done
