mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --iters 12"
timeout 300 $CMD > gpurun_out/plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_walk_lv" -c 2 -o gpurun_out/prof_walk $CMD > gpurun_out/ncu_walk.log 2>&1; echo "ncu walk rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_split|k_forward" -s 14 -c 2 -o gpurun_out/prof_split $CMD > gpurun_out/ncu_split.log 2>&1; echo "ncu split rc=$?"
