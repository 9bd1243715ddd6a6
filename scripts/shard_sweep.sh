#!/bin/bash
# Detached-shard timings of the 3D rank grids: rank 0 of an
# R-rank grid with Rv view groups, timed alone on one B200, for cfg3 (WAM,
# separable 3D Haar) and cfg5 (AM).  Output: gpurun_out/shard/<cfg>_R<R>_v<Rv>.json
set -u
out=${OUT:-gpurun_out/shard}
mkdir -p "$out"
for cfg in ${CFGS:-cfg3 cfg5}; do
  for R in ${RS:-2 4 8}; do
    for Rv in ${RVS:-1 2 4 8}; do
      [ $Rv -gt $R ] && continue
      timeout 600 python bench.py --config $cfg --shard $R --view-groups $Rv --steps ${STEPS:-3} --warmup 3 \
        > "$out/${cfg}_R${R}_v${Rv}.json" 2> "$out/${cfg}_R${R}_v${Rv}.err"
      echo "$cfg R=$R Rv=$Rv rc=$?"
    done
  done
done
