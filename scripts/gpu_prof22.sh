mkdir -p gpurun_out
CMD="python bench.py --config cfg2 --steps 1 --warmup 0 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1; echo "plain rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_walk" --csv --log-file gpurun_out/launches22.csv $CMD > gpurun_out/ncu22a.log 2>&1; echo "ncu-a rc=$?"
grep -E "k_walk" gpurun_out/launches22.csv | awk -F'","' '{print $5, $(NF)}' | head -20
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_walk_lv" -s 3 -c 1 -o gpurun_out/prof_walk22 $CMD > gpurun_out/ncu22.log 2>&1; echo "ncu rc=$?"
