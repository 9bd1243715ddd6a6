# Key histogram taken in the 2D walk's drain (k_key_hist skipped): GPU tests, cfg2 bench x3, launch list.
mkdir -p gpurun_out/s4h
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s4h/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s4h/pytest_gpu.log
for i in 1 2 3; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s4h/cfg2_$i.json 2> gpurun_out/s4h/cfg2_$i.err
python -c "
import json; d=json.load(open('gpurun_out/s4h/cfg2_$i.json')); print('run $i', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'ms', round(d['ms_per_step'],2), d['clocks']['sm_mhz'], 'expand', round(d['kernels']['per_step_ms']['expand'],2), d['final_objective'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/s4h/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s4h/ncu_ll.log 2>&1; echo "ncu-ll rc=$?"
python scripts/launches.py gpurun_out/s4h/launches_cfg2.csv > gpurun_out/s4h/launches_cfg2.txt; head -10 gpurun_out/s4h/launches_cfg2.txt
