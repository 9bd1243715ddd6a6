# ncu --set full of the slab kernels at a z-slab shard (cfg5 with nz = 8, P = 8) and at nz = 64 (default variant)
mkdir -p gpurun_out
for nz in 8 64; do
timeout 900 ncu --set full --clock-control none -f --import-source on -k regex:"k_fwd3s|k_back3s" -s 2 -c 2 -o /tmp/ncu5_nz$nz python bench.py --config cfg5 --nz $nz --steps 1 --warmup 0 --iters 2 --no-cpu-baseline > gpurun_out/ncu5_nz$nz.log 2>&1; echo "ncu nz$nz rc=$?"
ncu -i /tmp/ncu5_nz$nz.ncu-rep --page raw --csv > gpurun_out/ncu5_nz${nz}_raw.csv
ncu -i /tmp/ncu5_nz$nz.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/ncu5_nz${nz}_src.csv.gz
done
