# session 6 (container re-created, libwamgpu.so rebuilt from HEAD): confirm the suite, smoke and the contract line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s6_pytest.log 2>&1; tail -3 gpurun_out/s6_pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/s6_smoke.log 2>&1; tail -1 gpurun_out/s6_smoke.log
timeout 900 python bench.py > gpurun_out/s6_cfg4.log 2>&1; tail -1 gpurun_out/s6_cfg4.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print('cfg4',round(d['value'],3),round(d['e2e']['value'],3),d['clocks'],d['roofline'],d['cpu_baseline']['value'],d['gpu_launches'])"
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/s6_cfg4_reference.log 2>&1; tail -1 gpurun_out/s6_cfg4_reference.log | cut -c1-600
