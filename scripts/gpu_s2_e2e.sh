# streamed pinned boundary transfers + device transposes: full GPU tests, e2e at cfg5/cfg3/cfg2
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
for cfg in cfg5 cfg3 cfg2; do
timeout 900 python bench.py --config $cfg --steps 2 --warmup 2 --no-cpu-baseline > gpurun_out/e2e_$cfg.json 2>gpurun_out/e2e_$cfg.err
tail -1 gpurun_out/e2e_$cfg.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('$cfg it/s',round(d['value'],2),'e2e',round(d['e2e']['value'],2),d['e2e'],d['clocks']['sm_mhz'])"
done
