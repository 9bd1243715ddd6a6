# NF sweep of the ping-pong slab pipeline, then source-level ncu of the cfg4 split (final tree) and both 3D walks
mkdir -p gpurun_out/p2
run() { echo "== $1 $2 SLAB=$3"; WAMGPU_SLAB_VARIANT=$3 timeout 900 python scripts/cfg4_iters.py $1 $2 2>&1 | grep -v "^$" | tail -n 1; }
{ run cfg3 12 112; run cfg3 12 118; run cfg3 12 120; run cfg3 12 121; run cfg3 12 17; run cfg4 12 112; run cfg4 12 118; } > gpurun_out/p2/nf.log 2>&1
python - <<'PY'
import re
for l in open("gpurun_out/p2/nf.log"):
    l = l.strip()
    if l.startswith("=="): print(l); continue
    m = re.search(r"'fwd_ms': ([0-9.]+), 'back_ms': ([0-9.]+).*'fwd_launches': (\d+), 'back_launches': (\d+)", l)
    print("   fwd %.2f back %.2f ms/pass" % (float(m.group(1))/int(m.group(3)), float(m.group(2))/int(m.group(4))) if m else "   ? "+l[:200])
PY
python scripts/cfg4_iters.py cfg4 36 > gpurun_out/p2/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -f --import-source on -k regex:"k_split3h_e" -s 26 -c 1 -o /tmp/split4 python scripts/cfg4_iters.py cfg4 36 > gpurun_out/p2/split.log 2>&1; echo "ncu split rc=$?"
ncu -i /tmp/split4.ncu-rep --page raw --csv > gpurun_out/p2/split_raw.csv
ncu -i /tmp/split4.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/p2/split_src.csv.gz
timeout 900 ncu --set full --clock-control none -f --import-source on -k regex:"k_walk3h" -s 6 -c 2 -o /tmp/walk4 python scripts/cfg4_iters.py cfg4 36 > gpurun_out/p2/walk.log 2>&1; echo "ncu walk rc=$?"
ncu -i /tmp/walk4.ncu-rep --page raw --csv > gpurun_out/p2/walk_raw.csv
ncu -i /tmp/walk4.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/p2/walk_src.csv.gz
ls -la gpurun_out/p2; du -sh gpurun_out
