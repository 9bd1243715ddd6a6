# split with the two-stage prefetch + evict-first Psi loads (with and without ray bands); back NF variants at cfg4
mkdir -p gpurun_out/s2
timeout 900 python -m pytest tests/test_gpu_parity3d.py tests/test_gpu_sharded3d.py -x -q > gpurun_out/s2/pytest.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/s2/pytest.log
run() { echo "== $1 $2 SLAB=$3 SPLITBAND=$4"; WAMGPU_SLAB_VARIANT=$3 WAMGPU_SPLIT_BAND_MB=$4 timeout 900 python scripts/cfg4_iters.py $1 $2 2>&1 | grep -v "^$" | tail -n 2; }
{ run cfg3 30 112 0; run cfg3 30 112 48; run cfg4 40 112 0; run cfg4 40 118 48; run cfg4 40 120 24; run cfg4 40 121 96; } > gpurun_out/s2/ab.log 2>&1
python - <<'PY'
import re
for l in open("gpurun_out/s2/ab.log"):
    l = l.strip()
    if l.startswith("=="): print(l); continue
    m = re.search(r"'total_ms': ([0-9.]+), 'fwd_ms': ([0-9.]+), 'back_ms': ([0-9.]+), 'split_ms': ([0-9.]+).*'expand_ms': ([0-9.]+).*'fwd_launches': (\d+), 'back_launches': (\d+), 'split_launches': (\d+)", l)
    if m:
        t, f, b, s, e, nf, nb, ns = m.groups()
        print(f"   total {float(t):.0f} ms  fwd {float(f)/max(int(nf),1):.2f}  back {float(b)/max(int(nb),1):.2f}  split {float(s)/max(int(ns),1):.2f} ms/launch ({float(s):.0f} per run)  expand {float(e):.0f}")
    elif "objective" in l: print("   " + l[:110])
    else: print("   ?", l[:300])
PY
