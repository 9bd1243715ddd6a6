# on-the-fly TMA forward v2 (pipelined rings, integer h, CB retry): parity, then forward ms per pass
mkdir -p gpurun_out/tma2
timeout 600 python -m pytest tests/test_gpu_parity3d.py -x -q -k "on_the_fly" > gpurun_out/tma2/pytest.log 2>&1; rc=$?; echo "pytest rc=$rc"; tail -n 5 gpurun_out/tma2/pytest.log
[ $rc -ne 0 ] && exit 0
run() { echo "== $1 $2 FWD3T=$3 NF=$4"; WAMGPU_FWD3T=$3 WAMGPU_FWD3T_NF=$4 timeout 900 python scripts/cfg4_iters.py $1 $2 2>&1 | grep -v "^$" | tail -n 3; }
{
run cfg5 10 0 1; run cfg5 10 1 1; run cfg5 10 1 0; run cfg5 10 1 2
run cfg3 12 0 1; run cfg3 12 1 1; run cfg3 12 1 0
run cfg4 12 0 1; run cfg4 12 1 1; run cfg4 12 1 0
} > gpurun_out/tma2/ab.log 2>&1
grep -E "==|fwd_ms|rejected|Error" gpurun_out/tma2/ab.log | python -c "
import sys,re
for l in sys.stdin:
    l=l.strip()
    m=re.search(r\"'fwd_ms': ([0-9.]+).*'fwd_launches': (\d+)\", l)
    print(l[:100] if not m else '   fwd %.2f ms/pass over %s launches' % (float(m.group(1))/max(int(m.group(2)),1), m.group(2)))
"
