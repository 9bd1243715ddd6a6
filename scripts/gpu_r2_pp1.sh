# ping-pong slab pipeline (WAMGPU_SLAB_VARIANT=117) and banded split: parity on the 3D tests, then A/B
mkdir -p gpurun_out/pp1
WAMGPU_SLAB_VARIANT=117 WAMGPU_SPLIT_BAND_MB=0.01 timeout 900 python -m pytest tests/test_gpu_parity3d.py tests/test_gpu_sharded3d.py -x -q > gpurun_out/pp1/pytest_117.log 2>&1; echo "pytest(117, forced split bands) rc=$?"; tail -n 4 gpurun_out/pp1/pytest_117.log
timeout 900 python -m pytest tests/test_gpu_parity3d.py -x -q > gpurun_out/pp1/pytest_def.log 2>&1; echo "pytest(default) rc=$?"; tail -n 2 gpurun_out/pp1/pytest_def.log
run() { echo "== $1 $2 SLAB=$3 SPLITBAND=$4"; WAMGPU_SLAB_VARIANT=$3 WAMGPU_SPLIT_BAND_MB=$4 timeout 900 python scripts/cfg4_iters.py $1 $2 2>&1 | grep -v "^$" | tail -n 2; }
{
run cfg5 10 112 48; run cfg5 10 117 48
run cfg3 30 112 0; run cfg3 30 117 0; run cfg3 30 117 48; run cfg3 30 117 24
run cfg4 40 112 0; run cfg4 40 117 48; run cfg4 40 117 96; run cfg4 40 117 24
} > gpurun_out/pp1/ab.log 2>&1
python - <<'PY'
import re
for l in open("gpurun_out/pp1/ab.log"):
    l = l.strip()
    if l.startswith("=="): print(l); continue
    m = re.search(r"'total_ms': ([0-9.]+), 'fwd_ms': ([0-9.]+), 'back_ms': ([0-9.]+), 'split_ms': ([0-9.]+).*'expand_ms': ([0-9.]+).*'fwd_launches': (\d+), 'back_launches': (\d+), 'split_launches': (\d+)", l)
    if m:
        t, f, b, s, e, nf, nb, ns = m.groups()
        print(f"   total {float(t):.0f} ms  fwd {float(f)/max(int(nf),1):.2f}  back {float(b)/max(int(nb),1):.2f}  split {float(s)/max(int(ns),1):.2f} ms/launch  expand {float(e):.0f}")
    elif "objective" in l: print("   " + l[:110])
    else: print("   ?", l[:200])
PY
