# Split on the side stream, overlapped with the back projection (2D, one GPU):
# GPU tests, cfg2 bench A/B (overlap vs WAMGPU_SPLIT_OVERLAP=0), interleaved.
mkdir -p gpurun_out/s4o
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s4o/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s4o/pytest_gpu.log
for i in 1 2 3; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s4o/ovl_$i.json 2> gpurun_out/s4o/ovl_$i.err
WAMGPU_SPLIT_OVERLAP=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s4o/seq_$i.json 2> gpurun_out/s4o/seq_$i.err
done
python - <<'PY'
import json
for n in ["ovl_1","seq_1","ovl_2","seq_2","ovl_3","seq_3"]:
    try:
        d=json.load(open(f"gpurun_out/s4o/{n}.json"))
        print(n, round(d["value"],1), "e2e", round(d["e2e"]["value"],1), "ms", round(d["ms_per_step"],2), d["clocks"]["sm_mhz"], {k: round(v,2) for k,v in d["kernels"]["per_step_ms"].items()}, d["final_objective"])
    except Exception as e: print(n, "ERR", e)
PY
