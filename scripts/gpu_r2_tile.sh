# view x channel CTA tiles in the slab forward (WAMGPU_FWD_TILE = views per tile); new NF defaults
mkdir -p gpurun_out/tile
WAMGPU_FWD_TILE=4 timeout 900 python -m pytest tests/test_gpu_parity3d.py tests/test_gpu_sharded3d.py -x -q > gpurun_out/tile/pytest_t4.log 2>&1; echo "pytest(tile 4) rc=$?"; tail -n 3 gpurun_out/tile/pytest_t4.log
run() { echo "== $1 $2 TILE=$3"; WAMGPU_FWD_TILE=$3 timeout 900 python scripts/cfg4_iters.py $1 $2 2>&1 | grep -v "^$" | tail -n 2; }
{ run cfg5 10 0; run cfg5 10 4; run cfg3 12 0; run cfg3 12 2; run cfg3 12 4; run cfg3 12 8; run cfg4 12 0; run cfg4 12 2; run cfg4 12 4; run cfg4 12 8; } > gpurun_out/tile/ab.log 2>&1
python - <<'PY'
import re
for l in open("gpurun_out/tile/ab.log"):
    l = l.strip()
    if l.startswith("=="): print(l); continue
    m = re.search(r"'fwd_ms': ([0-9.]+), 'back_ms': ([0-9.]+).*'fwd_launches': (\d+), 'back_launches': (\d+)", l)
    if m: print("   fwd %.2f back %.2f ms/pass" % (float(m.group(1))/int(m.group(3)), float(m.group(2))/int(m.group(4))))
    elif "objective" in l: print("   " + l[:110])
    else: print("   ?", l[:300])
PY
