"""Wall time of each wam_expand call (synchronous at the ABI) vs its device
expand_ms, cfg2; prints host overhead per expansion."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1508_04458_b200 import configs
import paper_1508_04458_b200 as W

cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
g, I0, d = bench._inputs(cfg, W)
ctx = W.Context(0)
ctx.set_geometry(g)
if cfg["nz"] > 1:
    ctx.set_haar_dim(cfg["haar"])
ctx.set_data(d, I0)
for rep in range(2):
    t0 = time.perf_counter(); ctx.wam_init(cfg["L"]); t1 = time.perf_counter()
    print(f"init wall {1e3*(t1-t0):.2f} ms dev {ctx.timing()['total_ms']:.2f}")
    done = 0
    for ev in cfg["schedule"]:
        ctx.wam_iterate(ev - done); done = ev
        t0 = time.perf_counter(); n = ctx.wam_expand(0.1); t1 = time.perf_counter()
        t = ctx.timing()
        print(f"expand at {ev}: new {n} wall {1e3*(t1-t0):.2f} ms dev expand {t['expand_ms']:.2f} total {t['total_ms']:.2f} nnz_phi {t['split_nnz']}")
