mkdir -p gpurun_out
CMD="python bench.py --config cfg2 --steps 1 --warmup 0 --no-cpu-baseline"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_forward|k_back|k_split" -s 60 -c 3 -o gpurun_out/prof_fb24 $CMD > gpurun_out/ncu24.log 2>&1; echo "ncu rc=$?"
