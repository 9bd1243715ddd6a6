"""z-activity statistics of the separable-3D tree after each expansion (what a
split kernel that compacts active slice groups could skip).
  python scripts/tree_zstats.py cfg4"""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_1508_04458_b200 import configs
import paper_1508_04458_b200 as W

cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "cfg4")
g, I0, d = bench._inputs(cfg, W)
ctx = W.Context(0)
ctx.set_geometry(g)
ctx.set_haar_dim(cfg["haar"])
ctx.set_data(d, I0)
ctx.wam_init(cfg["L"])
nx, ny, nz, L = cfg["nx"], cfg["ny"], cfg["nz"], cfg["L"]
done = 0
for ev in cfg["schedule"]:
    ctx.wam_iterate(ev - done); done = ev
    n = ctx.wam_expand(0.1)
    t = ctx.tree()
    print(f"== expansion at {ev}: {n} new blocks, split entries {ctx.timing()['split_nnz']}")
    o = 0
    for l in range(1, L + 1):
        nk, hl, wl = nz >> l, ny >> l, nx >> l
        a = t[o:o + nk * hl * wl].reshape(nk, hl * wl).astype(bool); o += nk * hl * wl
        anyb = a.any(0)
        if not anyb.any():
            print(f"  level {l}: none"); continue
        al = a[:, anyb]                       # (nk, listed blocks)
        # slice groups of 8 slices: z-block k covers slices [k<<l, (k+1)<<l)
        sl = np.repeat(al, 1 << l, axis=0)    # per slice
        for G in (8, 16, 32):
            grp = sl.reshape(nz // G, G, -1).any(1)
            na = grp.sum(0)
            lpe = np.where(na > 0, 2 ** np.ceil(np.log2(np.maximum(na, 1))), 1)
            print(f"  level {l}: listed {anyb.sum()} of {anyb.size}, active z-blocks {al.mean():.3f}, "
                  f"groups of {G} slices active {grp.mean():.3f}, mean pow2 lanes/entry fraction {(lpe / (nz // G)).mean():.3f}")
ctx.close()
