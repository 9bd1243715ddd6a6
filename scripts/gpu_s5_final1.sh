# evidence at HEAD: full GPU suite, smoke, the contract bench line (cfg4, default flags) and the reference arm, cfg3/cfg2/cfg1/cfg5 lines,
# ncu launch list of the default bench command, ncu --set full of the split (final tree) and of a coarse forward + back
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -x -q > gpurun_out/s5_final_pytest.log 2>&1; tail -3 gpurun_out/s5_final_pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/s5_final_smoke.log 2>&1; tail -1 gpurun_out/s5_final_smoke.log
timeout 1800 python bench.py > gpurun_out/s5_final_cfg4.log 2>&1; tail -1 gpurun_out/s5_final_cfg4.log | cut -c1-600
timeout 1800 python bench.py --impl reference > gpurun_out/s5_final_cfg4_ref.log 2>&1; tail -1 gpurun_out/s5_final_cfg4_ref.log | cut -c1-400
for c in cfg3 cfg2 cfg1 cfg5; do
timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s5_final_$c.log 2>&1; tail -1 gpurun_out/s5_final_$c.log | cut -c1-200
done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/s5_launches_cfg4.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/s5_ncu_launches.log 2>&1; echo "launch list rc=$?"
gzip -f gpurun_out/s5_launches_cfg4.csv
timeout 900 ncu --set full --clock-control none -f --import-source on -k regex:"k_split3c" -s 26 -c 1 -o /tmp/split5 python scripts/cfg4_iters.py cfg4 36 > gpurun_out/s5_ncu_split.log 2>&1; echo "ncu split rc=$?"
ncu -i /tmp/split5.ncu-rep --page raw --csv > gpurun_out/s5_split3c_chunk_raw.csv
ncu -i /tmp/split5.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/s5_split3c_chunk_src.csv.gz
timeout 900 ncu --set full --clock-control none -f -k regex:"k_fwd3s|k_back3s|k_beer_z|k_qsum_z|k_g_expand_z|k_mu_coarse_z" -s 0 -c 40 -o /tmp/coarse5 python scripts/cfg4_iters.py cfg4 34 > gpurun_out/s5_ncu_coarse.log 2>&1; echo "ncu coarse rc=$?"
ncu -i /tmp/coarse5.ncu-rep --page raw --csv > gpurun_out/s5_coarse_raw.csv
gzip -f gpurun_out/s5_coarse_raw.csv
ls -la gpurun_out | tail -12
