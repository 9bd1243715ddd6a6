mkdir -p gpurun_out
CMD="python bench.py --config cfg2 --steps 1 --warmup 0 --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_fwd_patch|k_split" -s 60 -c 2 -o gpurun_out/prof_fwd31 $CMD > gpurun_out/ncu31.log 2>&1; echo "ncu rc=$?"
