# HEAD check: smoke, GPU tests, default bench line (with CPU baseline).
mkdir -p gpurun_out/head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/head/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/head/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/head/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/head/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/head/r04_cfg2.json 2> gpurun_out/head/r04_cfg2.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/head/r04_cfg2.json')); print(round(d['value'],1), d['e2e']['value'], d['roofline']['frac'], d['clocks'], d['cpu_baseline']['value'], d['gpu_launches'], round(d['ms_per_step'],2))"
