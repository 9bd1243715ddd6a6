mkdir -p gpurun_out
CMD="python bench.py --config cfg5 --steps 1 --warmup 0 --no-cpu-baseline --iters 2"
timeout 600 $CMD > gpurun_out/plain.log 2>&1; echo "plain rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_forward3|k_back3" -c 3 -o gpurun_out/prof_3d $CMD > gpurun_out/ncu_3d.log 2>&1; echo "ncu rc=$?"
