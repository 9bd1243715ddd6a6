# ncu --set full at cfg4 (WAM, 3D Haar L=4): slab forward/back, then the 3D split after 2 expansions
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none -f -k regex:"k_fwd3s|k_back3s" -s 2 -c 2 -o /tmp/ncu4_fb python bench.py --config cfg4 --steps 1 --warmup 0 --iters 2 --no-cpu-baseline > gpurun_out/ncu4_fb.log 2>&1; echo "ncu fb rc=$?"
ncu -i /tmp/ncu4_fb.ncu-rep --page raw --csv > gpurun_out/ncu4_fb_raw.csv
timeout 1500 ncu --set full --clock-control none -f -k regex:"k_split3h_e|k_walk3h" -s 20 -c 3 -o /tmp/ncu4_sp python bench.py --config cfg4 --steps 1 --warmup 0 --iters 20 --no-cpu-baseline > gpurun_out/ncu4_sp.log 2>&1; echo "ncu sp rc=$?"
ncu -i /tmp/ncu4_sp.ncu-rep --page raw --csv > gpurun_out/ncu4_sp_raw.csv
ncu -i /tmp/ncu4_sp.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/ncu4_sp_src.csv.gz
