"""Generates the BASELINE-size parity fixtures tests/golden/big_<cfg>.json
(committed) with the CPU oracle (test infrastructure; oracle/wam_oracle.cpp).

The GPU at cfg2-cfg5 finishes a whole reconstruction in well under a second,
but the oracle needs minutes to hours, so its trajectories are computed once
here and committed in compact form:

* inputs: SHA-256 of d and I0 (the GPU test regenerates them with the
  product's device simulator, whose counts equal the oracle's host generator,
  and checks the hashes);
* per oracle (``mirror`` = the fp32-storage oracle the GPU mirrors bit for bit;
  ``f64`` = reference precision): Z0 at init, the objective (I-divergence) of
  every iteration as float hex, the active-set / cumulative-update counters,
  and per scheduled expansion the number of newly active blocks, the SHA-256
  and per-level counts of the tree bytes, Z0, and the criterion tie margin
  (criterion values within 1e-5 * max of the 0.1 * max
  threshold, and the smallest distance);
* final state: a seeded CountSketch (K = 4096, fp32) of mu (and of beta for the
  f64 oracle) plus exact L2 norms, so the GPU's 1e-4 relative-L2 bar is checked without committing
  tens of MB of voxels (tests/wam_testutil.py count_sketch).

cfg4 is TRUNCATED: its oracle runs the first K iterations only (default 9 =
iterations 1-8, the first expansion after iteration 8, iteration 9), in the
slim CSR-only mode (the 1.87e9-entry in-plane matrix at 8 B per entry), and
only the fp32-mirror oracle: a reference-precision run at cfg4 does not fit
this 62 GB host.  The truncation is recorded in the fixture.

    python tests/golden/make_golden_big.py cfg2 [cfg3 cfg5 cfg4] [--threads N]
"""
import argparse
import base64
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import oracle as O  # noqa: E402
from paper_1508_04458_b200 import configs  # noqa: E402
from wam_testutil import count_sketch, tie_margin  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
TRUNC = {"cfg4": 9}
SLIM = {"cfg4"}
MIRROR_ONLY = {"cfg4"}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def b64(a):
    """fp32 sketch values (rounding noise ~6e-8 relative, far below the 1e-6 /
    1e-4 bars they check)"""
    return base64.b64encode(np.ascontiguousarray(a, np.float32).tobytes()).decode()


def hx(v):
    return float(v).hex()


def log(*a):
    print(f"[{time.strftime('%H:%M:%S')}]", *a, flush=True)


def tree_levels(tree, cfg):
    """Per-level active block counts of a tree byte array (get_tree layout)."""
    out, o = [], 0
    for lv in range(1, cfg["L"] + 1):
        n = (cfg["nx"] >> lv) * (cfg["ny"] >> lv) * ((cfg["nz"] >> lv) if cfg["haar"] == 3 and cfg["nz"] > 1 else 1)
        out.append(int(np.count_nonzero(tree[o:o + n])))
        o += n
    return out


def criterion(p, cfg):
    """The fp64 expansion criterion image the oracle's expand uses
    (image_of_beta(p, false), z-summed for the per-slice 2D model)."""
    beta = p.wam_get()["beta"]
    if cfg["nz"] > 1 and cfg["haar"] == 3:
        return O.idwt3(beta, cfg["nx"], cfg["ny"], cfg["nz"], cfg["L"])
    mu = O.idwt2(beta, cfg["nx"], cfg["ny"], cfg["L"])
    return mu.reshape(cfg["nz"], -1).sum(axis=0) if cfg["nz"] > 1 else mu


def run_wam(p, cfg, d, I0, J, beta_sketch):
    sched = [s for s in cfg["schedule"] if s < J]
    t0 = time.time()
    if cfg["nz"] > 1:
        p.set_haar_dim(cfg["haar"])
    p.wam_init(d, I0, cfg["L"])
    out = {"Z0_init": hx(p.wam_get()["Z0"]), "init_s": time.time() - t0, "objective": [], "active_set": [],
           "cum_updates": [], "expansions": []}
    log("  init", f"{out['init_s']:.1f}s Z0={p.wam_get()['Z0']}")
    done = 0
    for ev in sched + [J]:
        t1 = time.time()
        recs = p.wam_iterate(ev - done)
        out["objective"] += [hx(r[1]) for r in recs]
        out["active_set"] += [int(r[3]) for r in recs]
        out["cum_updates"] += [int(r[4]) for r in recs]
        log(f"  iterations {done + 1}..{ev}", f"{(time.time() - t1) / max(ev - done, 1):.1f}s/it",
            f"obj={recs[-1][1]!r}")
        done = ev
        if ev == J:
            break
        tm = tie_margin(criterion(p, cfg))
        t1 = time.time()
        n = p.wam_expand(0.1)
        tree = p.wam_tree()
        out["expansions"].append({"after_iter": ev, "newly": int(n), "tree_sha256": sha(tree),
                                  "tree_levels": tree_levels(tree, cfg), "Z0": hx(p.wam_get()["Z0"]),
                                  "tie": tm, "expand_s": time.time() - t1})
        log(f"  expand after {ev}: +{n} blocks, levels {tree_levels(tree, cfg)}, ties {tm}")
    g = p.wam_get()
    mu = g["mu"]
    out["final"] = {"mu_sketch": b64(count_sketch(mu)), "mu_norm": float(np.linalg.norm(mu)),
                    "mu_sum": float(mu.sum()), "beta_norm": float(np.linalg.norm(g["beta"])), "Z0": hx(g["Z0"]),
                    "counters": p.wam_counters()}
    if beta_sketch:
        out["final"]["beta_sketch"] = b64(count_sketch(g["beta"]))
    return out


def run_am(p, cfg, d, I0, J):
    t0 = time.time()
    p.am_init(d, I0)
    out = {"Z0_init": hx(p.am_get()["Z0"]), "init_s": time.time() - t0}
    t1 = time.time()
    recs = p.am_iterate(J)
    log(f"  {J} AM iterations", f"{(time.time() - t1) / J:.1f}s/it")
    out["objective"] = [hx(r[1]) for r in recs]
    mu = p.am_get()["mu"]
    out["final"] = {"mu_sketch": b64(count_sketch(mu)), "mu_norm": float(np.linalg.norm(mu)),
                    "mu_sum": float(mu.sum())}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--only", choices=["mirror", "f64"], default=None)
    a = ap.parse_args()
    for name in a.configs:
        cfg = configs.get(name)
        J = TRUNC.get(name, cfg["J"])
        og = O.make_geometry(**configs.geometry(cfg))
        path = os.path.join(HERE, f"big_{name}.json")
        res = json.load(open(path)) if os.path.exists(path) else {}
        res.update({"config": name, "algo": cfg["algo"], "J": J, "J_config": cfg["J"],
                    "truncated": J < cfg["J"], "schedule": [s for s in cfg["schedule"] if s < J],
                    "nx": cfg["nx"], "ny": cfg["ny"], "nz": cfg["nz"], "L": cfg["L"], "haar": cfg["haar"],
                    "sketch": {"K": 4096, "seed": "0x5EED5EED"}, "slim": name in SLIM})
        res.setdefault("oracles", {})
        kinds = [k for k in ("mirror", "f64") if not (k == "f64" and name in MIRROR_ONLY)]
        if a.only:
            kinds = [k for k in kinds if k == a.only]
        d = I0 = None
        for kind in kinds:
            log(name, kind, "building H")
            t0 = time.time()
            p = O.Problem(og, mirror=(kind == "mirror"), threads=a.threads, slim=name in SLIM)
            tb = time.time() - t0
            log(f"  H: nnz/slice {p.nnz}, {tb:.1f}s")
            if d is None:
                mu_true = O.rasterize(og, configs.phantom(cfg))
                I0 = configs.incident(cfg, p.M)
                d = p.simulate(mu_true, I0, cfg["seed"])
                del mu_true
                res["inputs"] = {"d_sha256": sha(d), "I0_sha256": sha(I0), "nnz_slice": int(p.nnz),
                                 "M_slice": int(p.M), "N_slice": int(p.N)}
                log("  inputs", res["inputs"])
            r = run_wam(p, cfg, d, I0, J, kind == "f64") if cfg["algo"] == "wam" else run_am(p, cfg, d, I0, J)
            r["build_s"] = tb
            r["threads"] = a.threads or os.cpu_count()
            res["oracles"][kind] = r
            del p
            with open(path, "w") as f:
                json.dump(res, f, indent=1)
            log("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
