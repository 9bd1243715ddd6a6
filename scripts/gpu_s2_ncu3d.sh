# ncu --set full of the current 3D slab kernels (cfg5, AM: forward + fused back/update)
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg5 --steps 1 --warmup 3 --iters 4 --no-cpu-baseline > gpurun_out/b5.json 2>gpurun_out/b5.err; echo "b5 rc=$?"; tail -c 400 gpurun_out/b5.json
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_forward3|k_back3" -s 2 -c 2 -o gpurun_out/ncu3d_s2 python bench.py --config cfg5 --steps 1 --warmup 0 --iters 2 --no-cpu-baseline > gpurun_out/ncu3d.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu3d.log
