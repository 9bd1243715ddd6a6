"""Shared helpers of the test suite (imported as a plain module)."""
import numpy as np


def problem_inputs(cfg_name, orc, W, mirror=False, threads=0):
    """Seeded inputs of a named config: (cfg, oracle problem, mu_true, I0, d)."""
    from paper_1508_04458_b200 import configs
    cfg = configs.get(cfg_name)
    og = orc.make_geometry(**configs.geometry(cfg))
    p = orc.Problem(og, mirror=mirror, threads=threads)
    mu_true = orc.rasterize(og, configs.phantom(cfg))
    I0 = configs.incident(cfg, p.M)
    d = p.simulate(mu_true, I0, cfg["seed"])
    return cfg, p, mu_true, I0, d


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
