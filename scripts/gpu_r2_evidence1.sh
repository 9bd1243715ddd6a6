# Round-2 evidence: ncu --set full of one banded forward pass + back + split at cfg4 (raw CSV only: the
# .ncu-rep is > 64 MiB); cfg2 view-shard projections; cfg2/cfg1 reference arm with 1 and all threads;
# cfg1/cfg2/cfg3/cfg5 bench lines.
mkdir -p gpurun_out/ev1
python scripts/cfg4_iters.py cfg4 34 > gpurun_out/ev1/cfg4_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none -k regex:"k_fwd3s_band|k_back3s|k_split3h_e" --launch-skip 290 -c 14 \
    -o /tmp/cfg4_pass -f python scripts/cfg4_iters.py cfg4 34 > gpurun_out/ev1/ncu.log 2>&1
echo "ncu rc=$?"; tail -n 2 gpurun_out/ev1/ncu.log
ncu -i /tmp/cfg4_pass.ncu-rep --page raw --csv > gpurun_out/ev1/cfg4_pass_raw.csv 2>/dev/null
python scripts/ncu_kv.py /tmp/cfg4_pass.ncu-rep > gpurun_out/ev1/ncu_cfg4_pass.txt 2>&1
for R in 2 4 8; do
  timeout 600 python bench.py --config cfg2 --shard $R --steps 5 --warmup 3 > gpurun_out/ev1/cfg2_R$R.json 2> gpurun_out/ev1/cfg2_R$R.err; echo "cfg2 shard $R rc=$?"
done
timeout 900 python bench.py --config cfg2 --steps 10 --warmup 3 > gpurun_out/ev1/r06_cfg2.json 2> gpurun_out/ev1/r06_cfg2.err; echo "cfg2 rc=$?"
timeout 900 python bench.py --impl reference --config cfg2 --steps 3 --warmup 3 > gpurun_out/ev1/r06_cfg2_reference.json 2> gpurun_out/ev1/ref2.err; echo "cfg2 ref rc=$?"
timeout 1200 python bench.py --impl reference --config cfg2 --cpu-threads 1 --steps 2 --warmup 3 > gpurun_out/ev1/r06_cfg2_reference_1thread.json 2> gpurun_out/ev1/ref2_1.err; echo "cfg2 ref 1 thread rc=$?"
timeout 900 python bench.py --impl reference --config cfg1 --cpu-threads 1 --steps 5 --warmup 3 > gpurun_out/ev1/r06_cfg1_reference_1thread.json 2> gpurun_out/ev1/ref1_1.err; echo "cfg1 ref 1 thread rc=$?"
for cfg in cfg1 cfg3 cfg5; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 > gpurun_out/ev1/r06_$cfg.json 2> gpurun_out/ev1/r06_$cfg.err; echo "$cfg rc=$?"
done
lscpu > gpurun_out/ev1/lscpu.txt
du -sh gpurun_out
