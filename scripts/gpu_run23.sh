mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 400 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --config cfg2 > gpurun_out/b_cfg2.log 2>&1
tail -1 gpurun_out/b_cfg2.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernels'];print('cfg2',round(d['value'],2),k.get('per_step_ms'))"
CMD="python bench.py --config cfg2 --steps 1 --warmup 0 --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_walk|Onesweep" --csv --log-file gpurun_out/launches23.csv $CMD > gpurun_out/ncu23a.log 2>&1; echo "ncu-a rc=$?"
python scripts/launches.py gpurun_out/launches23.csv
