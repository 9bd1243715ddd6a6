"""cfg4 wavelet-AM through the C-ABI for a given number of iterations (the
first H-path forward/back are iteration 9's, after the expansion at 8): the
target command of the cfg4 ncu captures (profiles/)."""
import sys
import time

sys.path.insert(0, ".")
import paper_1508_04458_b200 as W  # noqa: E402
from paper_1508_04458_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = configs.get(name)
g = configs.geometry(cfg, W.Geometry)
mu = W.rasterize(g, configs.phantom(cfg))
I0 = configs.incident(cfg, cfg["views"] * cfg["detectors"])
d = W.simulate_device(g, mu, I0, cfg["seed"])
c = W.Context(0)
c.set_geometry(g)
if cfg["algo"] == "wam":
    c.set_haar_dim(cfg["haar"])
c.set_data(d, I0)
c.set_kernel_timing(True)
t0 = time.time()
if cfg["algo"] == "wam":
    c.wam_init(cfg["L"])
    r = c.wam_run(iters, [s for s in cfg["schedule"] if s < iters], 0.1)
else:
    c.am_init()
    r = c.am_iterate(iters)
t = c.timing()
print(name, iters, "iterations", time.time() - t0, "s; last objective", r[-1]["objective"])
print({k: round(v, 3) if isinstance(v, float) else v for k, v in t.items()})
