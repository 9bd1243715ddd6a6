# ncu --set full of the 2D expansion walk (cfg2) and the 3D walk (cfg3)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -f --import-source on -k regex:"k_walk_lv" -s 1 -c 2 -o /tmp/ncu_walk2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_walk2.log 2>&1; echo "ncu walk2 rc=$?"
ncu -i /tmp/ncu_walk2.ncu-rep --page raw --csv > gpurun_out/ncu_walk2_raw.csv
ncu -i /tmp/ncu_walk2.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/ncu_walk2_src.csv.gz
timeout 900 ncu --set full --clock-control none -f --import-source on -k regex:"k_walk3h" -s 2 -c 2 -o /tmp/ncu_walk3 python bench.py --config cfg3 --steps 1 --warmup 0 --iters 16 --no-cpu-baseline > gpurun_out/ncu_walk3.log 2>&1; echo "ncu walk3 rc=$?"
ncu -i /tmp/ncu_walk3.ncu-rep --page raw --csv > gpurun_out/ncu_walk3_raw.csv
