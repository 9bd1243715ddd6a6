"""Generates tests/golden/golden.json (committed).

* ref_H: system matrices built by the UNMODIFIED reference headers
  (oracle/_ref/libwamref.so <- /root/reference/proj/include, build_system_matrix
  projector.hpp:126 and trace_ray for the pinned arc rays): nnz + SHA-256 of the
  CSR arrays.  Needs /root/reference at generation time only.
* tiny_*: the f64 (reference-precision) oracle trajectories of the `tiny`
  config: AM and wavelet-AM objectives per iteration, active-tree bitmaps after
  each expansion, Z0, and the final image (fp32) - the fixtures the GPU parity
  tests also check against.

    python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_1508_04458_b200 import configs  # noqa: E402

REF_GEOMS = {
    "parallel_16": (0, 16, 16, 1.0, 12, 24, 1.0),
    "fan_flat_32": (1, 32, 32, 1.0, 45, 48, 1.37),
    "fan_flat_64": (1, 64, 64, 0.5, 60, 96, 0.71),
}


def sha(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    out = {"_doc": __doc__.strip().splitlines()[0], "ref_H": {}}
    for name, (beam, nx, ny, vox, V, D, sp) in REF_GEOMS.items():
        r = O.RefMatrix.build(beam, nx, ny, 1, vox, V, D, sp, 500.0, 1000.0)
        rp, ci, v = r.csr()
        out["ref_H"][name] = dict(beam=beam, nx=nx, ny=ny, voxel=vox, views=V, detectors=D, spacing=sp,
                                  nnz=int(r.nnz), sha256=sha(rp, ci, v), row_sum_max=float(
                                      max(O.reflib().ref_row_sum(r.h, y) for y in range(r.M))))
    for name in ("tiny", "cfg1"):
        cfg = configs.get(name)
        p = O.Problem(O.make_geometry(**configs.geometry(cfg)))
        r = O.RefMatrix.from_rays(cfg["nx"], cfg["ny"], cfg["voxel"], p.rays())
        rp, ci, v = r.csr()
        out["ref_H"]["arc_" + name] = dict(config=name, nnz=int(r.nnz), sha256=sha(rp, ci, v))
    # tiny trajectories (f64 oracle)
    cfg = configs.get("tiny")
    og = O.make_geometry(**configs.geometry(cfg))
    p = O.Problem(og)
    mu_true = O.rasterize(og, configs.phantom(cfg))
    I0 = configs.incident(cfg, p.M)
    d = p.simulate(mu_true, I0, cfg["seed"])
    out["tiny_data_sha256"] = sha(d)
    p.am_init(d, I0)
    am = p.am_iterate(cfg["J"])
    out["tiny_am"] = dict(objective=[r[1] for r in am], Z0=p.am_get()["Z0"],
                          mu=p.am_get()["mu"].astype(np.float32).tolist())
    p.wam_init(d, I0, cfg["L"])
    objs, trees, z0s, done = [], [], [p.wam_get()["Z0"]], 0
    for ev in cfg["schedule"] + [cfg["J"]]:
        objs += [r[1] for r in p.wam_iterate(ev - done)]
        done = ev
        if ev == cfg["J"]:
            break
        p.wam_expand(0.1)
        trees.append(p.wam_tree().tobytes().hex())
        z0s.append(p.wam_get()["Z0"])
    out["tiny_wam"] = dict(L=cfg["L"], J=cfg["J"], schedule=cfg["schedule"], objective=objs, trees=trees, Z0=z0s,
                           counters=p.wam_counters(), mu=p.wam_get()["mu"].astype(np.float32).tolist())
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
