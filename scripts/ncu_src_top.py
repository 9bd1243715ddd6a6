"""Top SASS instructions by stall samples from an ncu --page source --csv export
(first kernel in the file), with the stall-reason columns that dominate.
usage: python scripts/ncu_src_top.py src.csv[.gz] [N]"""
import csv
import gzip
import io
import sys

f = sys.argv[1]
raw = gzip.open(f, "rt").read() if f.endswith(".gz") else open(f).read()
lines = raw.splitlines()
# the export repeats a "Kernel Name" line + header per kernel; take the first block
blocks, cur = [], None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = [ln]
        blocks.append(cur)
    elif cur is not None:
        cur.append(ln)
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for b in blocks:
    name = b[0].split(",", 1)[1][:90]
    rows = list(csv.reader(io.StringIO("\n".join(b[1:]))))
    hdr = rows[0]
    data = rows[1:]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or h.endswith("(All Samples)") and "Warp Stall" not in h]
    tot = sum(float(r[iS] or 0) for r in data)
    print("==", name, "total samples", tot)
    # per-opcode totals
    ops = {}
    for r in data:
        op = r[1].strip().split()[0] if r[1].strip() else "?"
        if op.startswith("@"):
            op = r[1].strip().split()[1]
        op = op.split(".")[0]
        ops[op] = ops.get(op, 0) + float(r[iS] or 0)
    print("   by opcode:", ", ".join(f"{k}={100*v/tot:.1f}%" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:12]))
    data.sort(key=lambda r: -float(r[iS] or 0))
    for r in data[:N]:
        print(f"   {100*float(r[iS])/tot:5.1f}%  {r[1].strip()[:70]}")
