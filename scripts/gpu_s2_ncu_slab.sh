# ncu --set full of slab variants (raw CSV exported on the box; reports removed: gpurun_out <= 64 MiB)
mkdir -p gpurun_out
for v in ${VARS:-1 9}; do
WAMGPU_SLAB_VARIANT=$v timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_forward3|k_back3|k_fwd3s|k_back3s" -s 2 -c 2 -o /tmp/ncu3d_v$v python bench.py --config ${CFG:-cfg5} --steps 1 --warmup 0 --iters 2 --no-cpu-baseline > gpurun_out/ncu3d_v$v.log 2>&1; echo "ncu v$v rc=$?"
ncu -i /tmp/ncu3d_v$v.ncu-rep --page raw --csv > gpurun_out/ncu3d_v${v}_raw.csv
ncu -i /tmp/ncu3d_v$v.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu3d_v${v}_src.csv 2>/dev/null
gzip -f gpurun_out/ncu3d_v${v}_src.csv
done
ls -la gpurun_out
