mkdir -p gpurun_out
CMD="python bench.py --config cfg2 --steps 1 --warmup 0 --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_fwd_c2" -s 30 -c 1 -o gpurun_out/prof_c2 $CMD > gpurun_out/ncu34.log 2>&1; echo "ncu rc=$?"
