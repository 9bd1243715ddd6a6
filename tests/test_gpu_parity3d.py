"""GPU parity of the axial 3D stack (nz > 1 slices sharing one in-plane system
matrix, geometry.hpp:17-20; pin P2) against the CPU oracle:
slab forward/back, the AM baseline and the wavelet AM with per-slice 2D Haar
and the z-summed expansion criterion.  `small3d` has 40
slices, exercising partially filled lane slabs (2 slices per lane, masked);
`tiny3d` / `tiny3d16` / `tiny3d24` use the slab strides 8, 16 and 32 (8 pad
slices) of z-slab shards."""
import numpy as np
import pytest

from wam_testutil import problem_inputs, rel_l2

pytestmark = pytest.mark.gpu
TOL_F64, TOL_MIRROR = 1e-4, 1e-6


def _ctx(W, cfg):
    from paper_1508_04458_b200 import configs
    c = W.Context(0)
    c.set_geometry(configs.geometry(cfg, W.Geometry))
    return c


@pytest.mark.parametrize("name", ["tiny3d", "tiny3d16", "tiny3d24", "small3d"])
def test_slab_forward_back_vs_mirror(wam, orc, name):
    cfg, p, mu_true, I0, d = problem_inputs(name, orc, wam, mirror=True)
    c = _ctx(wam, cfg)
    mu32 = mu_true.astype(np.float32).astype(np.float64)
    l_gpu, l_orc = c.forward_project(mu_true), p.forward_project(mu32)
    assert l_gpu.shape == l_orc.shape and rel_l2(l_gpu, l_orc) < 1e-14
    w = (I0 * np.exp(-l_orc)).astype(np.float32).astype(np.float64)
    assert rel_l2(c.back_project(w), p.back_project(w)) < 1e-14
    rng = np.random.default_rng(2)
    x = rng.standard_normal(p.N * p.nz).astype(np.float32).astype(np.float64)
    y = rng.standard_normal(p.M * p.nz).astype(np.float32).astype(np.float64)
    Hx, Hty = c.forward_project(x), c.back_project(y)
    assert abs(Hx @ y - x @ Hty) <= 1e-12 * np.linalg.norm(Hx) * np.linalg.norm(y)


@pytest.mark.parametrize("name", ["tiny3d", "small3d"])
def test_am3d_parity(wam, orc, name):
    cfg, p64, _, I0, d = problem_inputs(name, orc, wam)
    p32 = orc.Problem(p64.geom, mirror=True)
    c = _ctx(wam, cfg)
    c.set_data(d, I0)
    c.am_init()
    p64.am_init(d, I0)
    p32.am_init(d, I0)
    J = cfg["J"]
    og = np.array([r["objective"] for r in c.am_iterate(J)])
    o64 = [r[1] for r in p64.am_iterate(J)]
    o32 = [r[1] for r in p32.am_iterate(J)]
    assert rel_l2(og, o64) < TOL_F64 and rel_l2(og, o32) < TOL_MIRROR
    assert rel_l2(c.image(), p64.am_get()["mu"]) < TOL_F64
    assert rel_l2(c.image(), p32.am_get()["mu"]) < TOL_MIRROR
    assert all(b <= a * (1 + 1e-6) for a, b in zip(og, og[1:]))


@pytest.mark.parametrize("name", ["tiny3d", "small3d"])
def test_wam3d_parity_tree_bit_exact(wam, orc, name):
    cfg, p64, _, I0, d = problem_inputs(name, orc, wam)
    p32 = orc.Problem(p64.geom, mirror=True)
    L, J, sched = cfg["L"], cfg["J"], cfg["schedule"]
    c = _ctx(wam, cfg)
    c.set_data(d, I0)
    c.wam_init(L)
    p64.wam_init(d, I0, L)
    p32.wam_init(d, I0, L)
    assert c.scalars()["Z0"] == p32.wam_get()["Z0"]
    assert rel_l2(c.stats()[0], p32.wam_stats()[0]) < 1e-12
    og, o64, o32, done = [], [], [], 0
    for ev in sched + [J]:
        og += [r["objective"] for r in c.wam_iterate(ev - done)]
        o64 += [r[1] for r in p64.wam_iterate(ev - done)]
        o32 += [r[1] for r in p32.wam_iterate(ev - done)]
        done = ev
        if ev == J:
            break
        assert c.wam_expand(0.1) == p32.wam_expand(0.1)
        p64.wam_expand(0.1)
        assert np.array_equal(c.tree(), p32.wam_tree()) and np.array_equal(c.tree(), p64.wam_tree())
        assert c.scalars()["Z0"] == p32.wam_get()["Z0"]
    assert rel_l2(og, o64) < TOL_F64 and rel_l2(og, o32) < TOL_MIRROR
    assert rel_l2(c.image(), p64.wam_get()["mu"]) < TOL_F64
    assert rel_l2(c.image(), p32.wam_get()["mu"]) < TOL_MIRROR
    s, cnt = c.scalars(), p32.wam_counters()
    assert (s["active_set"], s["cum_updates"], s["degenerate"]) == (cnt["active_set"], cnt["cum_updates"],
                                                                      cnt["degenerate"])
    _, bp, bm = c.stats()
    _, bp32, bm32 = p32.wam_stats()
    assert rel_l2(bm, bm32) < TOL_MIRROR and rel_l2(bp, bp32) < TOL_MIRROR


@pytest.mark.parametrize("name", ["tiny3d", "tiny3d16", "tiny3d24", "tiny3d64", "small3d"])
def test_wam3d_separable_haar_parity(wam, orc, name):
    """Separable 3D Haar model (pin P3): octree tree bit-exact vs both oracles
    after every expansion, Z0 bit-exact vs the mirror, mu / I-div within bars."""
    cfg, p64, _, I0, d = problem_inputs(name, orc, wam)
    p32 = orc.Problem(p64.geom, mirror=True)
    L, J, sched = cfg["L"], cfg["J"], cfg["schedule"]
    c = _ctx(wam, cfg)
    c.set_haar_dim(3)
    c.set_data(d, I0)
    c.wam_init(L)
    for p in (p64, p32):
        p.set_haar_dim(3)
        p.wam_init(d, I0, L)
    assert c.scalars()["Z0"] == p32.wam_get()["Z0"]
    assert rel_l2(c.stats()[0], p32.wam_stats()[0]) < 1e-12
    og, o64, o32, done = [], [], [], 0
    for ev in sched + [J]:
        og += [r["objective"] for r in c.wam_iterate(ev - done)]
        o64 += [r[1] for r in p64.wam_iterate(ev - done)]
        o32 += [r[1] for r in p32.wam_iterate(ev - done)]
        done = ev
        if ev == J:
            break
        assert c.wam_expand(0.1) == p32.wam_expand(0.1)
        p64.wam_expand(0.1)
        assert np.array_equal(c.tree(), p32.wam_tree()) and np.array_equal(c.tree(), p64.wam_tree())
        assert c.scalars()["Z0"] == p32.wam_get()["Z0"]
        assert np.array_equal(c.z_rows(), p32.wam_z0_rows())
    assert rel_l2(og, o64) < TOL_F64 and rel_l2(og, o32) < TOL_MIRROR
    assert rel_l2(c.image(), p64.wam_get()["mu"]) < TOL_F64
    assert rel_l2(c.image(), p32.wam_get()["mu"]) < TOL_MIRROR
    s, cnt = c.scalars(), p32.wam_counters()
    assert (s["active_set"], s["cum_updates"], s["degenerate"]) == (cnt["active_set"], cnt["cum_updates"],
                                                                      cnt["degenerate"])
    _, bp, bm = c.stats()
    _, bp32, bm32 = p32.wam_stats()
    assert rel_l2(bm, bm32) < TOL_MIRROR and rel_l2(bp, bp32) < TOL_MIRROR


@pytest.mark.parametrize("root", ["phi_a", "coarse"])
@pytest.mark.parametrize("name", ["tiny3d16", "small3d"])
def test_root_only_iterations_use_phi_a_3d(wam, orc, name, root, monkeypatch):
    """Separable 3D Haar with only the roots active: the iterations run over the
    in-plane approximation columns (kernels_phi.cuh, 3D part; WAMGPU_COARSE_ROOT=0)
    or, by default, over the 2^L-coarsened matrix on z-groups (kernels3c.cuh),
    within the mirror bars, and the first expansion still matches the oracle
    bit-exactly."""
    monkeypatch.setenv("WAMGPU_COARSE_ROOT", "0" if root == "phi_a" else "1")
    cfg, p64, _, I0, d = problem_inputs(name, orc, wam)
    p32 = orc.Problem(p64.geom, mirror=True)
    c = _ctx(wam, cfg)
    c.set_haar_dim(3)
    c.set_data(d, I0)
    c.wam_init(cfg["L"])
    p32.set_haar_dim(3)
    p32.wam_init(d, I0, cfg["L"])
    n = cfg["schedule"][0]
    og = [r["objective"] for r in c.wam_iterate(n)]
    t = c.timing()
    if root == "phi_a":
        assert t["phi_launches"] == n and t["fwd_launches"] == 0 and t["back_launches"] == 0
    else:
        assert t["phi_launches"] == 0 and t["fwd_launches"] == 0 and t["back_launches"] == 0
        assert t["coarse_fwd_launches"] == n and t["coarse_back_launches"] == n
    assert rel_l2(og, [r[1] for r in p32.wam_iterate(n)]) < TOL_MIRROR
    assert rel_l2(c.image(), p32.wam_get()["mu"]) < TOL_MIRROR
    assert c.wam_expand(0.1) == p32.wam_expand(0.1)
    assert np.array_equal(c.tree(), p32.wam_tree())
    og2 = [r["objective"] for r in c.wam_iterate(2)]
    assert c.timing()["phi_launches"] == 0
    assert rel_l2(og2, [r[1] for r in p32.wam_iterate(2)]) < TOL_MIRROR


@pytest.mark.parametrize("name", ["tiny3d16", "small3d"])
def test_banded_forward(wam, orc, name, monkeypatch):
    """The banded 3D forward (k_fwd3s_band: image rows in bands whose mu stays
    L2-resident, per-ray band segments summed in band order; the cfg4 path) is
    forced on small stacks with a tiny band size: forward projection and the
    separable-Haar WAM run agree with the unbanded forward and the oracles."""
    cfg, p32, mu_true, I0, d = problem_inputs(name, orc, wam, mirror=True)
    out = {}
    for mb in ("0", "0.004"):
        monkeypatch.setenv("WAMGPU_FWD_BAND_MB", mb)
        c = _ctx(wam, cfg)
        l = c.forward_project(mu_true)
        c.set_haar_dim(3)
        c.set_data(d, I0)
        c.wam_init(cfg["L"])
        r = c.wam_run(cfg["J"], cfg["schedule"], 0.1)
        out[mb] = (l, [x["objective"] for x in r], c.tree(), c.image())
        c.close()
    (l0, o0, t0, m0), (l1, o1, t1, m1) = out["0"], out["0.004"]
    assert rel_l2(l1, l0) < 1e-14
    assert rel_l2(l1, p32.forward_project(mu_true.astype(np.float32).astype(np.float64))) < 1e-14
    assert rel_l2(o1, o0) < 1e-12 and np.array_equal(t1, t0) and rel_l2(m1, m0) < 1e-9
    p32.set_haar_dim(3)
    p32.wam_init(d, I0, cfg["L"])
    ro = p32.wam_run(cfg["J"], cfg["schedule"], 0.1)
    assert np.array_equal(t1, p32.wam_tree())
    assert rel_l2(o1, [x[1] for x in ro]) < TOL_MIRROR


@pytest.mark.parametrize("name", ["tiny3d24", "small3d", "tiny3d64"])
def test_on_the_fly_tma_forward(wam, orc, name):
    """The on-the-fly 3D forward (kernels3t.cuh k_fwd3t: rays re-traced every
    pass with the device Siddon tracer, image tiles staged by TMA, north_star
    item (2)) against the stored-matrix slab SpMM and the oracle: the same fp32
    h and the same ray-order fp64 sums, so line integrals are BIT-identical,
    and so are q, mu and the tree of a separable-Haar WAM run (only the order
    of the objective's partial sums differs).  Ragged bundles: 60 / 72 views
    (groups of 8), 96 channels (groups of 64), 24 / 40 slices (chunks of 32)."""
    cfg, p32, mu_true, I0, d = problem_inputs(name, orc, wam, mirror=True)
    rng = np.random.default_rng(5)
    x = rng.standard_normal(mu_true.size).astype(np.float32).astype(np.float64)   # signed values
    out = {}
    for kind in (0, 1):
        c = _ctx(wam, cfg)
        c.set_projector(kind)
        l, lx = c.forward_project(mu_true), c.forward_project(x)
        assert c.projector() == (2 if kind else 0), "on-the-fly projector rejected its bundle geometry"
        c.set_haar_dim(3)
        c.set_data(d, I0)
        c.wam_init(cfg["L"])
        r = c.wam_run(cfg["J"], cfg["schedule"], 0.1)
        out[kind] = (l, lx, [v["objective"] for v in r], c.tree(), c.image(), c.q())
        assert c.projector() == (2 if kind else 0)
        c.close()
    (l0, x0, o0, t0, m0, q0), (l1, x1, o1, t1, m1, q1) = out[0], out[1]
    assert np.array_equal(l1, l0) and np.array_equal(x1, x0)
    assert rel_l2(l1, p32.forward_project(mu_true.astype(np.float32).astype(np.float64))) < 1e-14
    assert np.array_equal(t1, t0) and np.array_equal(m1, m0) and np.array_equal(q1, q0)
    assert rel_l2(o1, o0) < 1e-13


@pytest.mark.parametrize("name", ["tiny3d16", "small3d", "tiny3d64"])
def test_split_variants_agree(wam, orc, name, monkeypatch):
    """The opt-in 3D split k_split3z (WAMGPU_SPLIT_VARIANT=7: a lane per ACTIVE
    z-block, the oracle's qlo/qhi/qall formulation, one product per z-high
    coefficient) against the default k_split3h_e (every z-block of a listed
    block, both products): same tree, b- equal to rounding (the two sum in
    different but fixed orders), and b- within the mirror bar."""
    cfg, p32, _, I0, d = problem_inputs(name, orc, wam, mirror=True)
    out = {}
    for v in ("7", "0"):
        monkeypatch.setenv("WAMGPU_SPLIT_VARIANT", v)
        c = _ctx(wam, cfg)
        c.set_haar_dim(3)
        c.set_data(d, I0)
        c.wam_init(cfg["L"])
        r = c.wam_run(cfg["J"], cfg["schedule"], 0.1)
        out[v] = ([x["objective"] for x in r], c.tree(), c.image(), c.stats()[2])
        c.close()
    (o0, t0, m0, b0), (o6, t6, m6, b6) = out["7"], out["0"]
    assert np.array_equal(t0, t6)
    assert rel_l2(b0, b6) < 1e-13 and rel_l2(o0, o6) < 1e-12 and rel_l2(m0, m6) < 1e-6
    p32.set_haar_dim(3)
    p32.wam_init(d, I0, cfg["L"])
    p32.wam_run(cfg["J"], cfg["schedule"], 0.1)
    assert np.array_equal(t0, p32.wam_tree())
    assert rel_l2(b0, p32.wam_stats()[2]) < 1e-6
