# Incremental 3D active count: 3D GPU tests, cfg3 bench, cfg3 R=8 detached shard.
mkdir -p gpurun_out/s4c
timeout 1200 python -m pytest tests/test_gpu_parity3d.py tests/test_gpu_sharded3d.py tests/test_gpu_placement.py -q -x > gpurun_out/s4c/pytest_3d.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/s4c/pytest_3d.log
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 > gpurun_out/s4c/cfg3.json 2> gpurun_out/s4c/cfg3.err; echo "cfg3 rc=$?"
timeout 600 python bench.py --config cfg3 --shard 8 --view-groups 8 --steps 3 --warmup 3 > gpurun_out/s4c/cfg3_R8_v8.json 2> gpurun_out/s4c/cfg3_R8_v8.err; echo "shard rc=$?"
python - <<'PY'
import json
for n in ["cfg3","cfg3_R8_v8"]:
    try:
        d=json.load(open(f"gpurun_out/s4c/{n}.json"))
        print(n, round(d["value"],2), d["ms_per_step"], (d.get("shard") or {}).get("projected_ms_per_step"), d["clocks"], {k: round(v,2) for k,v in d["kernels"]["per_step_ms"].items()}, d["final_objective"])
    except Exception as e: print(n, "ERR", e)
PY
