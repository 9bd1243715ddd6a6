mkdir -p gpurun_out
CMD="python bench.py --config cfg2 --steps 1 --warmup 0 --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_walk_lv" -s 3 -c 1 -o gpurun_out/prof_walk30 $CMD > gpurun_out/ncu30.log 2>&1; echo "ncu rc=$?"
