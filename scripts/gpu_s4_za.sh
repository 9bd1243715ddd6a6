# zA cached across wam_init calls: GPU tests, cfg2 bench x2, cfg1, cfg3.
mkdir -p gpurun_out/s4z
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s4z/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s4z/pytest_gpu.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s4z/cfg2_$i.json 2> gpurun_out/s4z/cfg2_$i.err; echo "cfg2 rc=$?"
done
timeout 600 python bench.py --config cfg1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s4z/cfg1.json 2> gpurun_out/s4z/cfg1.err; echo "cfg1 rc=$?"
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s4z/cfg3.json 2> gpurun_out/s4z/cfg3.err; echo "cfg3 rc=$?"
python - <<'PY'
import json
for n in ["cfg2_1","cfg2_2","cfg1","cfg3"]:
    try:
        d=json.load(open(f"gpurun_out/s4z/{n}.json"))
        print(n, round(d["value"],1), "e2e", round(d["e2e"]["value"],1), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], {k: round(v,2) for k,v in d["kernels"]["per_step_ms"].items()}, d["final_objective"], d["gpu_launches"])
    except Exception as e: print(n, "ERR", e)
PY
