# ncu --set full (source-level) of the 2D expansion walk k_walk_lv (cfg2, 4th expansion)
# and of the 3D Z walk k_walk3h<1,3> (cfg3, 3rd expansion); reports stay in /tmp,
# raw + source CSVs come back.
mkdir -p gpurun_out/s4n
timeout 900 ncu --set full --clock-control none -f --import-source on -k regex:"k_walk_lv" -s 3 -c 1 -o /tmp/walk2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/s4n/walk2.log 2>&1; echo "ncu walk2 rc=$?"
ncu -i /tmp/walk2.ncu-rep --page raw --csv > gpurun_out/s4n/walk2_raw.csv
ncu -i /tmp/walk2.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/s4n/walk2_src.csv.gz
timeout 900 ncu --set full --clock-control none -f --import-source on -k regex:"k_walk3h" -s 4 -c 1 -o /tmp/walk3 python bench.py --config cfg3 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/s4n/walk3.log 2>&1; echo "ncu walk3 rc=$?"
ncu -i /tmp/walk3.ncu-rep --page raw --csv > gpurun_out/s4n/walk3_raw.csv
ncu -i /tmp/walk3.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/s4n/walk3_src.csv.gz
ls -la gpurun_out/s4n
