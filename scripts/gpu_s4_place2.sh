# Plain-atomic counting placement: placement tests, GPU tests, cfg2 bench
# (2 runs + the radix-sort path), launch list; cfg3 detached-shard projections
# (views-only grids) after the 3D Phi_A change.
mkdir -p gpurun_out/s4q gpurun_out/s4q/shard
timeout 900 python -m pytest tests/test_gpu_placement.py -q -x > gpurun_out/s4q/place_test.log 2>&1; echo "place test rc=$?"; tail -3 gpurun_out/s4q/place_test.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s4q/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s4q/pytest_gpu.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s4q/place_$i.json 2> gpurun_out/s4q/place_$i.err; echo "place rc=$?"
done
WAMGPU_PHI_SORT=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s4q/sort_1.json 2> gpurun_out/s4q/sort_1.err; echo "sort rc=$?"
python - <<'PY'
import json
for n in ["place_1","place_2","sort_1"]:
    try:
        d=json.load(open(f"gpurun_out/s4q/{n}.json"))
        print(n, round(d["value"],1), "e2e", round(d["e2e"]["value"],1), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], {k: round(v,2) for k,v in d["kernels"]["per_step_ms"].items()}, d["final_objective"])
    except Exception as e: print(n, "ERR", e)
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/s4q/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s4q/ncu_ll.log 2>&1; echo "ncu-ll rc=$?"
python scripts/launches.py gpurun_out/s4q/launches_cfg2.csv > gpurun_out/s4q/launches_cfg2.txt; head -12 gpurun_out/s4q/launches_cfg2.txt
for R in 2 4 8; do
timeout 600 python bench.py --config cfg3 --shard $R --view-groups $R --steps 3 --warmup 3 > gpurun_out/s4q/shard/cfg3_R${R}_v${R}.json 2> gpurun_out/s4q/shard/cfg3_R${R}_v${R}.err; echo "shard R=$R rc=$?"
done
