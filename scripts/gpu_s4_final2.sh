# Final cfg2 evidence at HEAD (after the split overlap): smoke, default bench with CPU baseline, launch list.
mkdir -p gpurun_out/end2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/end2/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/end2/smoke.log
timeout 900 python bench.py > gpurun_out/end2/r04_cfg2.json 2> gpurun_out/end2/r04_cfg2.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/end2/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/end2/ncu_ll.log 2>&1; echo "ncu-ll rc=$?"
python scripts/launches.py gpurun_out/end2/launches_cfg2.csv > gpurun_out/end2/launches_cfg2.txt; head -12 gpurun_out/end2/launches_cfg2.txt
python -c "
import json; d=json.load(open('gpurun_out/end2/r04_cfg2.json')); print(round(d['value'],1), d['e2e'], d['roofline']['frac'], d['clocks'], d['cpu_baseline'], d['gpu_launches'], {k: round(v,2) for k,v in d['kernels']['per_step_ms'].items()})"
