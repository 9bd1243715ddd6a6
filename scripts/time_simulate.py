"""Wall time of the host and device simulators (simulate_counts) per config."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import paper_1508_04458_b200 as W
from paper_1508_04458_b200 import configs

for name in sys.argv[1:]:
    cfg = configs.get(name)
    g = configs.geometry(cfg, W.Geometry)
    mu = W.rasterize(g, configs.phantom(cfg))
    I0 = configs.incident(cfg, cfg["views"] * cfg["detectors"])
    W.simulate_device(configs.geometry(configs.get("tiny"), W.Geometry),
                      W.rasterize(configs.geometry(configs.get("tiny"), W.Geometry), configs.phantom(configs.get("tiny"))),
                      configs.incident(configs.get("tiny"), 60 * 64), 1)   # context warm-up
    t0 = time.perf_counter(); dd = W.simulate_device(g, mu, I0, cfg["seed"]); td = time.perf_counter() - t0
    t0 = time.perf_counter(); dh = W.simulate(g, mu, I0, cfg["seed"]); th = time.perf_counter() - t0
    print(f"{name}: rays x slices {I0.size}, device {td:.2f} s, host {th:.2f} s ({__import__('os').cpu_count()} threads), "
          f"identical counts: {np.array_equal(dd, dh)}", flush=True)
