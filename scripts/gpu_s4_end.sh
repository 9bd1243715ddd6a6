# Session-4 closing evidence at HEAD: smoke, all GPU tests, default bench (cfg2 +
# CPU baseline), reference arm, cfg1/cfg3/cfg5/cfg4 lines, cfg3 R=8 shard, cfg2 launch list.
mkdir -p gpurun_out/end
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/end/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/end/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/end/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/end/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/end/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/end/r04_cfg2.json 2> gpurun_out/end/r04_cfg2.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/end/r04_cfg2_reference.json 2> gpurun_out/end/ref.err; echo "ref rc=$?"
timeout 900 python bench.py --config cfg1 --steps 3 --warmup 3 > gpurun_out/end/r04_cfg1.json 2> gpurun_out/end/r04_cfg1.err; echo "cfg1 rc=$?"
for cfg in cfg3 cfg5; do
timeout 900 python bench.py --config $cfg --steps 3 --warmup 3 > gpurun_out/end/r04_$cfg.json 2> gpurun_out/end/r04_$cfg.err; echo "$cfg rc=$?"
done
timeout 600 python bench.py --config cfg3 --shard 8 --view-groups 8 --steps 3 --warmup 3 > gpurun_out/end/cfg3_R8_v8.json 2> gpurun_out/end/cfg3_R8_v8.err; echo "shard rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/end/launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/end/ncu_ll.log 2>&1; echo "ncu-ll rc=$?"
python scripts/launches.py gpurun_out/end/launches_cfg2.csv > gpurun_out/end/launches_cfg2.txt
timeout 1500 python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/end/r04_cfg4.json 2> gpurun_out/end/r04_cfg4.err; echo "cfg4 rc=$?"
