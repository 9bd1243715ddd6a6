mkdir -p gpurun_out/guards
python - <<'PY' > gpurun_out/guards/script.py
import re
s = open("tests/test_gpu_guards.py").read()
body = s.split('SCRIPT = r"""')[1].split('"""')[0]
print(body % {"root": "/root/repo"})
PY
for g in 0 1; do
echo "== guard=$g banded"
WAMGPU_GUARD=$g WAMGPU_FWD_BAND_MB=0.004 timeout 150 python gpurun_out/guards/script.py 2>&1 | tail -n 12 | cut -c1-300
done
