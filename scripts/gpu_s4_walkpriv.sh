# Warp-private staging in the 2D expansion walk (nlev == 1): GPU tests, cfg2 bench x2, launch list.
mkdir -p gpurun_out/s4v
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s4v/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s4v/pytest_gpu.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s4v/cfg2_$i.json 2> gpurun_out/s4v/cfg2_$i.err; echo "cfg2 rc=$?"
done
python - <<'PY'
import json
for n in ["cfg2_1","cfg2_2"]:
    try:
        d=json.load(open(f"gpurun_out/s4v/{n}.json"))
        print(n, round(d["value"],1), "e2e", round(d["e2e"]["value"],1), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], {k: round(v,2) for k,v in d["kernels"]["per_step_ms"].items()}, d["final_objective"])
    except Exception as e: print(n, "ERR", e)
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/s4v/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s4v/ncu_ll.log 2>&1; echo "ncu-ll rc=$?"
python scripts/launches.py gpurun_out/s4v/launches_cfg2.csv > gpurun_out/s4v/launches_cfg2.txt; head -12 gpurun_out/s4v/launches_cfg2.txt
