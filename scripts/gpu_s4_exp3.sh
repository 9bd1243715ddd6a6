# Where the separable-3D expansion time goes (cfg3): host-traced phases of each
# wam_expand, and the cfg3 kernel launch list.
mkdir -p gpurun_out/s4e
WAMGPU_TRACE_HOST=1 timeout 900 python scripts/time_expand.py cfg3 > gpurun_out/s4e/trace_cfg3.log 2>&1; echo "trace rc=$?"
grep -v "^\[wamgpu\] *iter" gpurun_out/s4e/trace_cfg3.log | tail -60
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/s4e/launches_cfg3.csv python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/s4e/ncu_ll.log 2>&1; echo "ncu-ll rc=$?"
python scripts/launches.py gpurun_out/s4e/launches_cfg3.csv > gpurun_out/s4e/launches_cfg3.txt; head -30 gpurun_out/s4e/launches_cfg3.txt
