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


# ---------------------------------------------------------------- compact fingerprints
SKETCH_K = 4096
SKETCH_SEED = 0x5EED5EED


def _mix64(z):
    z = (z + np.uint64(0x9E3779B97F4A7C15))
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def count_sketch(x, K=SKETCH_K, seed=SKETCH_SEED, chunk=1 << 24):
    """CountSketch S x (K buckets, seeded splitmix64 hash and sign per index):
    E||S x||^2 = ||x||^2 with relative std ~ sqrt(2/K) (2% at K = 4096), and S is
    linear, so ||S a - S b|| / ||S b|| estimates rel_l2(a, b) without storing b.
    Deterministic: np.bincount sums in index order."""
    x = np.asarray(x, np.float64).ravel()
    out = np.zeros(K)
    with np.errstate(over="ignore"):
        for o in range(0, x.size, chunk):
            i = np.arange(o, min(o + chunk, x.size), dtype=np.uint64)
            h = _mix64(i ^ np.uint64(seed))
            b = (h & np.uint64(K - 1)).astype(np.int64)
            sg = ((h >> np.uint64(32)) & np.uint64(1)).astype(np.float64) * 2.0 - 1.0
            out += np.bincount(b, weights=sg * x[o:o + i.size], minlength=K)
    return out


def sketch_rel(x, ref_sketch):
    s = count_sketch(x, K=len(ref_sketch))
    r = np.asarray(ref_sketch, np.float64)
    return float(np.linalg.norm(s - r) / max(np.linalg.norm(r), 1e-300))


def tie_margin(crit, factor=0.1, rel=1e-5):
    """Expansion-criterion tie diagnostic: the number of
    criterion values within rel * max of the threshold factor * max, and the
    smallest |v - thr| / max."""
    crit = np.asarray(crit, np.float64)
    mx = float(crit.max())
    if not mx > 0:
        return {"max": mx, "thr": None, "ties": 0, "min_margin": None}
    thr = factor * mx
    dist = np.abs(crit - thr) / mx
    return {"max": mx, "thr": thr, "ties": int((dist < rel).sum()), "min_margin": float(dist.min())}
