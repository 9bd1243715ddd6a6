mkdir -p gpurun_out
( while true; do nvidia-smi --query-gpu=memory.used --format=csv,noheader >> gpurun_out/mem_cfg4.txt; sleep 2; done ) &
MP=$!
start=$(date +%s)
timeout 2400 python bench.py --config cfg4 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_cfg4.log 2> gpurun_out/bench_cfg4.err; echo "bench cfg4 rc=$? in $(( $(date +%s) - start )) s"
kill $MP
tail -1 gpurun_out/bench_cfg4.log | cut -c1-2500; tail -3 gpurun_out/bench_cfg4.err; sort -n gpurun_out/mem_cfg4.txt | tail -1
