mkdir -p gpurun_out
CMD="python bench.py --config cfg2 --steps 1 --warmup 0 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1; echo "plain rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches20.csv $CMD > gpurun_out/ncu20.log 2>&1; echo "ncu rc=$?"
python scripts/launches.py gpurun_out/launches20.csv | head -30
