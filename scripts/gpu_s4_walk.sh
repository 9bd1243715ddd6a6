# All-levels-per-thread expansion walk (k_walk_all) vs the warp-per-level
# k_walk_lv (WAMGPU_WALK_VARIANT=5): variant test, GPU tests, cfg2 bench A/B.
mkdir -p gpurun_out/s4w
timeout 600 python -m pytest tests/test_gpu_walk.py -q -x > gpurun_out/s4w/walk_test.log 2>&1; echo "walk test rc=$?"; tail -3 gpurun_out/s4w/walk_test.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s4w/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4w/pytest_gpu.log
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s4w/all_$i.json 2> gpurun_out/s4w/all_$i.err; echo "all rc=$?"
WAMGPU_WALK_VARIANT=5 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s4w/lv_$i.json 2> gpurun_out/s4w/lv_$i.err; echo "lv rc=$?"
done
python - <<'PY'
import json
for n in ["all_1","lv_1","all_2","lv_2"]:
    try:
        d=json.load(open(f"gpurun_out/s4w/{n}.json"))
        print(n, round(d["value"],1), "e2e", round(d["e2e"]["value"],1), {k: round(v,2) for k,v in d["kernels"]["per_step_ms"].items()}, d["tree"]["active_set_by_iteration"], d["final_objective"])
    except Exception as e: print(n, "ERR", e)
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/s4w/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s4w/ncu_ll.log 2>&1; echo "ncu-ll rc=$?"
python scripts/launches.py gpurun_out/s4w/launches_cfg2.csv > gpurun_out/s4w/launches_cfg2.txt; head -14 gpurun_out/s4w/launches_cfg2.txt
timeout 600 ncu --set full --clock-control none -f --import-source on -k regex:"k_walk_all" -s 3 -c 1 -o gpurun_out/s4w/ncu_walk python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/s4w/ncu_walk.log 2>&1; echo "ncu-walk rc=$?"
