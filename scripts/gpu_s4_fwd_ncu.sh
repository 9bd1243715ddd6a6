# cfg4 forward only (second try; the two-kernel capture left the forward with 6 of 39 passes)
python scripts/cfg4_iters.py cfg4 9 > gpurun_out/s4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_fwd3s" -c 1 \
    -o gpurun_out/s4_cfg4_fwd python scripts/cfg4_iters.py cfg4 9 > gpurun_out/s4_ncu.log 2>&1
echo rc=$?
tail -n 8 gpurun_out/s4_ncu.log
