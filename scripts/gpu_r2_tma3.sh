# on-the-fly TMA forward: cfg4 with the 32-channel retry; full ncu of one k_fwd3t launch at cfg5 (A/B evidence)
mkdir -p gpurun_out/tma3
run() { echo "== $1 $2 FWD3T=$3 NF=$4"; WAMGPU_FWD3T=$3 WAMGPU_FWD3T_NF=$4 timeout 900 python scripts/cfg4_iters.py $1 $2 2>&1 | grep -v "^$" | tail -n 3; }
{ run cfg4 12 1 0; run cfg4 12 1 1; } > gpurun_out/tma3/ab_cfg4.log 2>&1
cat gpurun_out/tma3/ab_cfg4.log | cut -c1-400
export WAMGPU_FWD3T=1 WAMGPU_FWD3T_NF=0
python scripts/cfg4_iters.py cfg5 2 > gpurun_out/tma3/plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fwd3t -c 1 -o gpurun_out/tma3/fwd3t_cfg5 -f python scripts/cfg4_iters.py cfg5 2 > gpurun_out/tma3/ncu.log 2>&1
echo "ncu rc=$?"; tail -n 3 gpurun_out/tma3/ncu.log; ls -la gpurun_out/tma3
