# cfg4: per-kernel times of a 10-iteration run (first H-path passes at iteration 9),
# then one ncu --set full capture of the slab forward and back kernels.
python scripts/cfg4_iters.py cfg4 10 > gpurun_out/s3_cfg4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_fwd3s|k_back3s" -c 2 \
    -o gpurun_out/s3_cfg4_slab python scripts/cfg4_iters.py cfg4 10 > gpurun_out/s3_ncu.log 2>&1
echo rc=$?
tail -5 gpurun_out/s3_cfg4_plain.log gpurun_out/s3_ncu.log
