# cfg3 views-only shards (R = 1, 2, 4, 8) and cfg4 (R = 1, 8) with the final build
mkdir -p gpurun_out/shard2
for R in 1 2 4 8; do
  timeout 600 python bench.py --config cfg3 --shard $R --view-groups $R --steps 3 --warmup 3 > gpurun_out/shard2/cfg3_R${R}_v$R.json 2> gpurun_out/shard2/cfg3_R$R.err; echo "cfg3 R=$R rc=$?"
done
for R in 1 2 4 8; do
  timeout 600 python bench.py --config cfg5 --shard $R --view-groups $R --steps 3 --warmup 3 > gpurun_out/shard2/cfg5_R${R}_v$R.json 2> gpurun_out/shard2/cfg5_R$R.err; echo "cfg5 R=$R rc=$?"
done
timeout 1500 python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/shard2/cfg4_R1_v1.json 2> gpurun_out/shard2/cfg4_R1.err; echo "cfg4 R=1 rc=$?"
timeout 1500 python bench.py --config cfg4 --shard 8 --view-groups 8 --steps 1 --warmup 3 > gpurun_out/shard2/cfg4_R8_v8.json 2> gpurun_out/shard2/cfg4_R8.err; echo "cfg4 R=8 rc=$?"
timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 > gpurun_out/shard2/r03_cfg3.json 2> gpurun_out/shard2/r03_cfg3.err; echo "cfg3 bench rc=$?"
