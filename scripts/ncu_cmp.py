"""Side-by-side key metrics of ncu raw-CSV exports (one column per kernel launch).
usage: python scripts/ncu_cmp.py a_raw.csv [b_raw.csv ...]"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors_srcunit_tex_op_read.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers"]
cols = []
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hdr = rows[0]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        d["_name"] = f.split("/")[-1][:12] + ":" + d.get("Kernel Name", "")[:22]
        stalls = []
        for h, v in d.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((h[34:-23], float(v)))
                except ValueError:
                    pass
        stalls.sort(key=lambda x: -x[1])
        d["_stalls"] = " ".join(f"{a}={b:.1f}" for a, b in stalls[:4])
        cols.append(d)
print("metric".ljust(60), " | ".join(c["_name"].ljust(36) for c in cols))
for k in KEYS:
    print(k[:60].ljust(60), " | ".join(str(c.get(k, "-"))[:36].ljust(36) for c in cols))
for c in cols:
    print(c["_name"], "stalls:", c["_stalls"])
