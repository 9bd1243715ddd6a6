# 3D emission walk with alternate level-1 emissions on two warps: 3D GPU tests, cfg3 bench, launch list.
mkdir -p gpurun_out/s4k
timeout 1200 python -m pytest tests/test_gpu_parity3d.py tests/test_gpu_sharded3d.py -q -x > gpurun_out/s4k/pytest_3d.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s4k/pytest_3d.log
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s4k/cfg3.json 2> gpurun_out/s4k/cfg3.err; echo "cfg3 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/s4k/cfg3.json')); print('cfg3', round(d['value'],2), d['ms_per_step'], {k: round(v,2) for k,v in d['kernels']['per_step_ms'].items()}, d['final_objective'])"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_walk3h|k_split3h|k_gather_psi|Onesweep" -c 400 --csv --log-file gpurun_out/s4k/launches_cfg3.csv python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s4k/ncu_ll.log 2>&1; echo "ncu-ll rc=$?"
python scripts/launches.py gpurun_out/s4k/launches_cfg3.csv > gpurun_out/s4k/launches_cfg3.txt; head -10 gpurun_out/s4k/launches_cfg3.txt
