"""Sharded axial 3D stacks on one GPU: R contexts joined as an in-process rank
group (wamgpu_set_comm_local, one host thread per rank), partitioned as an
Rv x Rz grid of view groups x z-slabs.  View
shards of a slab sum their partial back projections [H^T q || b-] (fp64) every
iteration; z-slabs exchange scalars only.  Every grid must reproduce the
unsharded run: the active tree bit-exactly after every expansion (the tree
of the unsharded run is itself bit-exact vs the oracle,
tests/test_gpu_parity3d.py), Z0 bit-exactly, the I-divergence trajectory and
mu within the mirror bar (the view-sharded g is summed in a different order)."""
import itertools
import threading

import numpy as np
import pytest

from wam_testutil import problem_inputs, rel_l2

pytestmark = pytest.mark.gpu
TOL = 1e-6
_key = itertools.count(1000)


def _slab_tree(tree, cfg, L, s0, nzl):
    """The z-slab [s0, s0+nzl) of a separable-3D tree (level l: (nz>>l, ny>>l, nx>>l))."""
    out, o = [], 0
    for l in range(1, L + 1):
        nb = (cfg["nx"] >> l) * (cfg["ny"] >> l)
        lv = tree[o:o + nb * (cfg["nz"] >> l)].reshape(cfg["nz"] >> l, nb)
        out.append(lv[s0 >> l:(s0 + nzl) >> l].ravel())
        o += nb * (cfg["nz"] >> l)
    return np.concatenate(out)


def _run(wam, cfg, I0, d, algo, haar, grid, sched):
    from paper_1508_04458_b200 import configs
    Rv, Rz = grid
    R = Rv * Rz
    key = next(_key)
    g = configs.geometry(cfg, wam.Geometry)
    ctxs = []
    for r in range(R):
        c = wam.Context(0)
        if R > 1:
            c.set_comm_local(key, r, R)
            c.set_partition(Rv)
        c.set_geometry(g)
        if algo == "wam" and cfg["nz"] > 1:
            c.set_haar_dim(haar)
        c.set_data(d, I0)
        ctxs.append(c)
    out = [None] * R
    errs = []
    J = cfg["J"]

    def work(r):
        c = ctxs[r]
        try:
            res = {"trees": [], "z0": []}
            if algo == "am":
                c.am_init()
                res["obj"] = [x["objective"] for x in c.am_iterate(J)]
            else:
                c.wam_init(cfg["L"])
                res["z0"].append(c.scalars()["Z0"])
                obj, done = [], 0
                for ev in sched + [J]:
                    obj += [x["objective"] for x in c.wam_iterate(ev - done)]
                    done = ev
                    if ev == J:
                        break
                    res.setdefault("newly", []).append(c.wam_expand(0.1))
                    res["trees"].append(c.tree())
                    res["z0"].append(c.scalars()["Z0"])
                res["obj"] = obj
            res["mu"] = c.image()
            res["part"] = c.partition()
            res["scal"] = c.scalars()
            out[r] = res
        except Exception as e:  # re-raised below
            errs.append(e)

    ths = [threading.Thread(target=work, args=(r,)) for r in range(R)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for c in ctxs:
        c.close()
    if errs:
        raise errs[0]
    return out


CASES = [
    ("tiny3d16", "am", 2, (2, 1)),
    ("tiny3d16", "am", 2, (2, 2)),
    ("tiny3d16", "am", 2, (3, 1)),          # 32 rows % 3: all-reduce + replicated update
    ("tiny3d16", "wam", 2, (3, 1)),
    ("tiny3d16", "wam", 2, (2, 2)),
    ("tiny3d16", "wam", 3, (2, 1)),
    ("tiny3d16", "wam", 3, (4, 1)),
    ("tiny3d16", "wam", 3, (2, 2)),
    ("tiny3d16", "wam", 3, (1, 2)),
    ("tiny3d24", "wam", 3, (3, 1)),         # 4 tile rows % 3: all-reduce + replicated update
    ("tiny", "wam", 2, (2, 1)),             # 2D view shards: all-reduce of [g || b-] (NCCL's path)
    ("tiny", "wam", 2, (3, 1)),
    ("tiny", "am", 2, (2, 1)),
]


@pytest.mark.parametrize("name,algo,haar,grid", CASES)
def test_sharded3d_matches_unsharded(wam, orc, name, algo, haar, grid):
    cfg, _, _, I0, d = problem_inputs(name, orc, wam)
    sched = cfg["schedule"]
    ref = _run(wam, cfg, I0, d, algo, haar, (1, 1), sched)[0]
    out = _run(wam, cfg, I0, d, algo, haar, grid, sched)
    Rv, Rz = grid
    N, L = cfg["nx"] * cfg["ny"], cfg["L"]
    mu = np.zeros(N * cfg["nz"])
    for r, res in enumerate(out):
        p = res["part"]
        assert (p["view_groups"], p["z_groups"]) == (Rv, Rz)
        s0, nzl = p["slab_begin"], p["slab_slices"]
        mu[s0 * N:(s0 + nzl) * N] = res["mu"][s0 * N:(s0 + nzl) * N]
        # every rank reports the global objective
        assert rel_l2(res["obj"], ref["obj"]) < TOL, f"rank {r}"
        assert res["obj"] == out[0]["obj"]
        if Rz == 1:   # slab-local counters: the whole stack here
            for k in ("cum_updates", "degenerate", "active_set"):
                assert res["scal"][k] == ref["scal"][k], (r, k)
        if algo == "wam":
            assert res["z0"] == ref["z0"], f"rank {r}: Z0 differs"
            for t, tref in zip(res["trees"], ref["trees"]):
                want = tref if haar == 2 else _slab_tree(tref, cfg, L, s0, nzl)
                assert np.array_equal(t, want), f"rank {r}: active tree differs"
    assert rel_l2(mu, ref["mu"]) < TOL
    # view shards of one slab hold the same (replicated) mu
    for a in range(len(out)):
        s0, nzl = out[a]["part"]["slab_begin"], out[a]["part"]["slab_slices"]
        sl = slice(s0 * N, (s0 + nzl) * N)
        for b in range(len(out)):
            if a // Rv == b // Rv:
                assert np.array_equal(out[a]["mu"][sl], out[b]["mu"][sl])


def test_detached_shard_runs_its_share(wam, orc):
    """A detached shard computes rank's share alone (timing hook): its matrix
    holds exactly its view rows and its slab, and it iterates without peers."""
    from paper_1508_04458_b200 import configs
    cfg, _, _, I0, d = problem_inputs("tiny3d16", orc, wam)
    g = configs.geometry(cfg, wam.Geometry)
    c = wam.Context(0)
    c.set_comm_local(-1, 1, 4)
    c.set_partition(2)
    c.set_geometry(g)
    p = c.partition()
    assert (p["view_groups"], p["z_groups"], p["slab_begin"], p["slab_slices"]) == (2, 2, 0, 8)
    V, D = cfg["views"], cfg["detectors"]
    assert (c.row0, c.row1) == (V // 2 * D, V * D)
    c.set_haar_dim(3)
    c.set_data(d, I0)
    c.wam_init(cfg["L"])
    recs = c.wam_run(4, [2], 0.1)
    assert len(recs) == 4 and all(np.isfinite(r["objective"]) for r in recs)
    c.close()


@pytest.mark.parametrize("name,haar", [("tiny", 2), ("tiny3d16", 2), ("tiny3d16", 3)])
def test_expand_with_replays_a_tree(wam, orc, name, haar):
    """wamgpu_wam_expand_with(+inf, tree): a second run that only replays the
    first run's trees reproduces its trajectory bit-exactly (same data, same
    tree, same kernels); a tree of the wrong size is a ContractError."""
    from paper_1508_04458_b200 import configs
    cfg, _, _, I0, d = problem_inputs(name, orc, wam)
    g = configs.geometry(cfg, wam.Geometry)
    runs = []
    trees = None
    for replay in (False, True):
        c = wam.Context(0)
        c.set_geometry(g)
        if cfg["nz"] > 1:
            c.set_haar_dim(haar)
        c.set_data(d, I0)
        c.wam_init(cfg["L"])
        obj, got, done = [], [], 0
        for k, ev in enumerate(cfg["schedule"] + [cfg["J"]]):
            obj += [r["objective"] for r in c.wam_iterate(ev - done)]
            done = ev
            if ev == cfg["J"]:
                break
            if replay:   # through the text manifest: resume a tree
                from paper_1508_04458_b200 import harness as H
                dims = (cfg["nx"], cfg["ny"], cfg["nz"], cfg["L"], haar if cfg["nz"] > 1 else 2)
                c.wam_expand(float("inf"), add_tree=H.parse_manifest(H.tree_manifest(trees[k], *dims), *dims))
            else:
                c.wam_expand(0.1)
            got.append(c.tree())
        if replay:
            with pytest.raises(wam.ContractError):
                c.wam_expand(0.1, add_tree=np.zeros(3, np.uint8))
        runs.append((obj, got, c.image()))
        trees = got
        c.close()
    (o1, t1, m1), (o2, t2, m2) = runs
    assert all(np.array_equal(a, b) for a, b in zip(t1, t2))
    assert o1 == o2 and np.array_equal(m1, m2)
