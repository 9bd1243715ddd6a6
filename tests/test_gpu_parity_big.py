"""GPU parity at the BASELINE sizes (north_star: "the active tree bit-exact at
every iteration, mu and the I-divergence trajectory within 1e-4 relative L2 on
all five configs").

* cfg2, cfg3, cfg5 and cfg4 (truncated, see below) against the committed
  oracle fixtures tests/golden/big_<cfg>.json (tests/golden/make_golden_big.py):
  the GPU run regenerates its inputs with the product's device simulator and
  first checks their SHA-256 against the fixture's (same seeded counts as the
  oracle's host generator), then compares
    - the tree after every scheduled expansion: SHA-256 equal to the fp32-mirror
      oracle's (bit-exact), and to the reference-precision oracle's whenever the
      two oracles agree (the fixture records the criterion tie margin);
    - the number of newly active blocks, Z0 at init and after every expansion
      (bit-exact vs the mirror, 1e-6 vs f64), the final active-set,
      cumulative-update and degenerate counters (exact vs the mirror);
    - the objective (I-divergence) of every iteration: 1e-4 relative L2 vs the
      f64 oracle (north_star), 1e-6 vs the mirror;
    - mu (and beta) through a seeded CountSketch: 1e-4 vs f64, 1e-6 vs mirror.
  cfg4 covers iterations 1-9 (root-only iterations 1-8, the first expansion,
  iteration 9 over the new tree) against the fp32-mirror oracle only: a full
  40-iteration run of the oracle at cfg4 takes hours, and the
  reference-precision oracle does not fit the 62 GB host that generates the
  fixtures.
* cfg2 additionally LIVE: both oracles run on the GPU box's host cores beside
  the GPU (full 50 iterations, 4 expansions), tree bit-exact after every
  expansion, Z(y) per ray and b- bit-exact vs the mirror at the end.
"""
import base64
import hashlib
import json
import os

import numpy as np
import pytest

from wam_testutil import rel_l2, sketch_rel, tie_margin

pytestmark = pytest.mark.gpu

TOL_F64, TOL_MIRROR = 1e-4, 1e-6
HERE = os.path.dirname(os.path.abspath(__file__))


def _fixture(name):
    path = os.path.join(HERE, "golden", f"big_{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    return json.load(open(path))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _sk(s):
    return np.frombuffer(base64.b64decode(s), np.float32).astype(np.float64)


def _inputs(W, cfg):
    from paper_1508_04458_b200 import configs
    g = configs.geometry(cfg, W.Geometry)
    mu_true = W.rasterize(g, configs.phantom(cfg))
    I0 = configs.incident(cfg, cfg["views"] * cfg["detectors"])
    d = W.simulate_device(g, mu_true, I0, cfg["seed"])
    return g, I0, d


def _ctx(W, cfg, g, I0, d):
    c = W.Context(0)
    c.set_geometry(g)
    if cfg["nz"] > 1 and cfg["algo"] == "wam":
        c.set_haar_dim(cfg["haar"])
    c.set_data(d, I0)
    return c


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4"])
def test_wam_against_baseline_size_fixture(wam, name):
    from paper_1508_04458_b200 import configs
    G = _fixture(name)
    cfg = configs.get(name)
    g, I0, d = _inputs(wam, cfg)
    assert _sha(d) == G["inputs"]["d_sha256"] and _sha(I0) == G["inputs"]["I0_sha256"]
    c = _ctx(wam, cfg, g, I0, d)
    assert c.nnz == G["inputs"]["nnz_slice"]
    mir = G["oracles"]["mirror"]
    f64 = G["oracles"].get("f64")
    c.wam_init(cfg["L"])
    assert c.scalars()["Z0"] == float.fromhex(mir["Z0_init"])
    objs, done = [], 0
    report = []
    for k, ev in enumerate(G["schedule"] + [G["J"]]):
        recs = c.wam_iterate(ev - done)
        objs += [r["objective"] for r in recs]
        done = ev
        if ev == G["J"]:
            break
        crit_tie = None
        if cfg["nz"] == 1:
            crit_tie = tie_margin(c.image())      # the GPU's own criterion image (fp32 mu)
        n = c.wam_expand(0.1)
        e = mir["expansions"][k]
        t = c.tree()
        report.append((ev, n, e["tie"], crit_tie))
        assert n == e["newly"], f"expansion after {ev}: {n} newly active blocks, mirror oracle {e['newly']}"
        assert _sha(t) == e["tree_sha256"], f"tree differs from the mirror oracle after iteration {ev}"
        assert c.scalars()["Z0"] == float.fromhex(e["Z0"])
        if f64 is not None:
            ef = f64["expansions"][k]
            if ef["tree_sha256"] == e["tree_sha256"]:
                assert _sha(t) == ef["tree_sha256"]
            else:   # the two oracles themselves differ: a criterion tie (recorded margin)
                print(f"{name}: f64 and mirror oracle trees differ after {ev}: tie {ef['tie']}")
            assert abs(c.scalars()["Z0"] - float.fromhex(ef["Z0"])) <= 1e-6 * float.fromhex(ef["Z0"])
    print(f"{name} expansions (after, newly, oracle tie margin, GPU criterion tie margin): {report}")
    og = np.array(objs)
    assert rel_l2(og, [float.fromhex(x) for x in mir["objective"]]) < TOL_MIRROR
    assert [r for r in mir["active_set"]][-1] == c.scalars()["active_set"]
    s, cnt = c.scalars(), mir["final"]["counters"]
    assert (s["active_set"], s["cum_updates"], s["degenerate"]) == \
        (cnt["active_set"], cnt["cum_updates"], cnt["degenerate"])
    mu = c.image()
    assert sketch_rel(mu, _sk(mir["final"]["mu_sketch"])) < TOL_MIRROR
    assert abs(np.linalg.norm(mu) - mir["final"]["mu_norm"]) <= TOL_MIRROR * mir["final"]["mu_norm"]
    if f64 is not None:
        assert rel_l2(og, [float.fromhex(x) for x in f64["objective"]]) < TOL_F64
        assert sketch_rel(mu, _sk(f64["final"]["mu_sketch"])) < TOL_F64
        assert sketch_rel(c.beta(), _sk(f64["final"]["beta_sketch"])) < TOL_F64
    assert all(b <= a * (1 + 1e-6) for a, b in zip(og, og[1:]))


def test_am_cfg5_against_fixture(wam):
    from paper_1508_04458_b200 import configs
    G = _fixture("cfg5")
    cfg = configs.get("cfg5")
    g, I0, d = _inputs(wam, cfg)
    assert _sha(d) == G["inputs"]["d_sha256"]
    c = _ctx(wam, cfg, g, I0, d)
    c.am_init()
    assert c.scalars()["Z0"] == float.fromhex(G["oracles"]["mirror"]["Z0_init"])
    og = np.array([r["objective"] for r in c.am_iterate(G["J"])])
    mu = c.image()
    for kind, tol in (("mirror", TOL_MIRROR), ("f64", TOL_F64)):
        o = G["oracles"].get(kind)
        if o is None:
            continue
        assert rel_l2(og, [float.fromhex(x) for x in o["objective"]]) < tol
        assert sketch_rel(mu, _sk(o["final"]["mu_sketch"])) < tol
    assert all(b <= a * (1 + 1e-6) for a, b in zip(og, og[1:]))


def test_cfg2_live_against_both_oracles(wam, orc):
    """The full cfg2 schedule on the GPU and, in the same process, on both CPU
    oracles (all host cores): tree bit-exact vs both after every expansion,
    Z0 and Z(y) bit-exact vs the mirror, I-div and mu within the bars."""
    from paper_1508_04458_b200 import configs
    cfg = configs.get("cfg2")
    g, I0, d = _inputs(wam, cfg)
    og_ = orc.make_geometry(**configs.geometry(cfg))
    p64 = orc.Problem(og_, mirror=False)
    p32 = orc.Problem(og_, mirror=True)
    c = _ctx(wam, cfg, g, I0, d)
    L, J, sched = cfg["L"], cfg["J"], cfg["schedule"]
    c.wam_init(L)
    p64.wam_init(d, I0, L)
    p32.wam_init(d, I0, L)
    assert c.scalars()["Z0"] == p32.wam_get()["Z0"]
    obj_g, obj64, obj32, done = [], [], [], 0
    for ev in sched + [J]:
        n = ev - done
        obj_g += [r["objective"] for r in c.wam_iterate(n)]
        obj64 += [r[1] for r in p64.wam_iterate(n)]
        obj32 += [r[1] for r in p32.wam_iterate(n)]
        done = ev
        if ev == J:
            break
        tie = tie_margin(p64.wam_get()["mu"])
        n_g, n_32, n_64 = c.wam_expand(0.1), p32.wam_expand(0.1), p64.wam_expand(0.1)
        print(f"cfg2 expansion after {ev}: GPU {n_g}, mirror {n_32}, f64 {n_64}, tie margin {tie}")
        assert n_g == n_32
        t = c.tree()
        assert np.array_equal(t, p32.wam_tree()), f"tree differs from the mirror oracle after iteration {ev}"
        assert np.array_equal(t, p64.wam_tree()), f"tree differs from the f64 oracle after iteration {ev}"
        assert c.scalars()["Z0"] == p32.wam_get()["Z0"]
    assert np.array_equal(c.z_rows(), p32.wam_z0_rows())
    assert rel_l2(obj_g, obj64) < TOL_F64 and rel_l2(obj_g, obj32) < TOL_MIRROR
    assert rel_l2(c.image(), p64.wam_get()["mu"]) < TOL_F64
    assert rel_l2(c.image(), p32.wam_get()["mu"]) < TOL_MIRROR
    assert rel_l2(c.beta(), p64.wam_get()["beta"]) < TOL_F64
    s, cnt = c.scalars(), p32.wam_counters()
    assert (s["active_set"], s["cum_updates"], s["degenerate"]) == \
        (cnt["active_set"], cnt["cum_updates"], cnt["degenerate"])
    _, bp_g, bm_g = c.stats()
    _, bp32, bm32 = p32.wam_stats()
    assert rel_l2(bm_g, bm32) < TOL_MIRROR and rel_l2(bp_g, bp32) < TOL_MIRROR
