# Counting placement of the Phi^- batch (replaces the radix sort): GPU tests,
# cfg2 bench A/B against the radix sort (WAMGPU_PHI_SORT=1), launch list.
mkdir -p gpurun_out/s4p
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s4p/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4p/pytest_gpu.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s4p/place_$i.json 2> gpurun_out/s4p/place_$i.err; echo "place rc=$?"
WAMGPU_PHI_SORT=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s4p/sort_$i.json 2> gpurun_out/s4p/sort_$i.err; echo "sort rc=$?"
done
python - <<'PY'
import json
for n in ["place_1","sort_1","place_2","sort_2"]:
    d=json.load(open(f"gpurun_out/s4p/{n}.json"))
    print(n, round(d["value"],1), "e2e", round(d["e2e"]["value"],1), {k: round(v,2) for k,v in d["kernels"]["per_step_ms"].items()}, d["tree"]["active_set_by_iteration"], d["final_objective"])
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/s4p/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s4p/ncu_ll.log 2>&1; echo "ncu-ll rc=$?"
python scripts/launches.py gpurun_out/s4p/launches_cfg2.csv > gpurun_out/s4p/launches_cfg2.txt; head -24 gpurun_out/s4p/launches_cfg2.txt
