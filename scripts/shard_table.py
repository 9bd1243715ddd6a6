"""Summarise detached-shard bench lines (scripts/shard_sweep.sh) into projected
strong-scaling efficiencies E(R) = T1 / (R * T_R)."""
import glob
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/shard"
rows, base = [], {}
for f in sorted(glob.glob(os.path.join(d, "*.json"))):
    try:
        L = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        print(f, "no result")
        continue
    cfg, R, v = os.path.basename(f)[:-5].split("_")
    R, v = int(R[1:]), int(v[1:])
    proj = L.get("shard", {}).get("projected_ms_per_step", L["ms_per_step"])
    if R == 1:
        base[cfg] = L["ms_per_step"]
    rows.append((cfg, R, v, L, proj))
print("| config | R | Rv x Rz | shard ms/run | modelled comm ms/run | projected ms/run | E(R) | fwd | back | split | update | expand | active set (last) |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for cfg, R, v, L, proj in sorted(rows, key=lambda r: (r[0], r[1], -r[2])):
    k = L["kernels"]["per_step_ms"]
    E = base[cfg] / (R * proj) if cfg in base else float("nan")
    print(f"| {cfg} | {R} | {v} x {R // v} | {L['ms_per_step']:.1f} | {proj - L['ms_per_step']:.1f} | {proj:.1f} | "
          f"{E:.2f} | {k['forward']:.0f} | {k['back']:.0f} | {k['split']:.0f} | {k['update']:.0f} | {k['expand']:.0f} | "
          f"{L['tree']['active_set_by_iteration'][-1]} |")
