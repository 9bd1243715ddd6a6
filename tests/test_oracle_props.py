"""Property tests the SPEC requires, run on the CPU oracle:
adjoint identity, monotone I-divergence, reduction equivalence, Z0 validity,
expansion-oracle set equality, adaptivity economy, noiseless consistency,
determinism.  Together with the KATs these pin the oracle."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from wam_testutil import problem_inputs


def _geom(n=32, V=60, D=64, vox=4.0):
    W = n * vox
    return O.make_geometry(n, n, 1, vox, V, D, beam=2, dgamma=2 * math.asin(W / 1000.0) / D)


def test_adjoint_identity():  # SPEC.md:80, 101, acceptance 4
    p = O.Problem(_geom(32, 40, 48), threads=2)
    rng = np.random.default_rng(3)
    for _ in range(100):
        x = rng.standard_normal(p.N)
        y = rng.standard_normal(p.M)
        Hx = p.forward_project(x)
        Hty = p.back_project(y)
        lhs, rhs = Hx @ y, x @ Hty
        assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(Hx) * np.linalg.norm(y)


@pytest.mark.parametrize("mirror", [0, 1])
def test_am_monotone(mirror):
    _, p, _, I0, d = problem_inputs("tiny", O, None, mirror=mirror)
    p.am_init(d, I0)
    obj = [r[1] for r in p.am_iterate(100)]
    for a, b in zip(obj, obj[1:]):
        assert b <= a * (1 + 1e-9)


@pytest.mark.parametrize("mirror", [0, 1])
def test_wam_monotone_with_expansions(mirror):
    cfg, p, _, I0, d = problem_inputs("tiny", O, None, mirror=mirror)
    p.wam_init(d, I0, cfg["L"])
    recs = p.wam_run(60, [10, 20, 30], 0.1)
    obj = [r[1] for r in recs]
    for a, b in zip(obj, obj[1:]):
        assert b <= a * (1 + 1e-9)
    assert recs[-1][3] > recs[0][3]           # the tree grew


def test_reduction_equivalence():  # SPEC.md:377, 393, acceptance 2: 16x16, 20 iterations, 1e-10
    g = _geom(16, 30, 32, 8.0)
    p = O.Problem(g)
    mu_t = O.rasterize(g, [dict(kind=0, cx=0, cy=0, cz=0, ax=40, ay=30, az=1, angle=0.2, value=0.02)])
    I0 = np.full(p.M, 1e5)
    d = p.simulate(mu_t, I0, 5)
    a = O.Problem(g)
    a.am_init(d, I0)
    a.am_set_clamp(0)
    w = O.Problem(g)
    w.wam_init(d, I0, 0)                      # Omega = I, full set
    assert abs(a.am_get()["Z0"] - w.wam_get()["Z0"]) <= 1e-12 * a.am_get()["Z0"]
    for _ in range(20):
        a.am_iterate(1)
        w.wam_iterate(1)
        assert np.abs(a.am_get()["mu"] - w.wam_get()["beta"]).max() <= 1e-10


def test_z0_validity_and_definition():  # SPEC.md:396, acceptance 5, Eq. 1.61
    cfg, p, _, I0, d = problem_inputs("tiny", O, None)
    p.wam_init(d, I0, cfg["L"])
    p.wam_run(12, [4, 8], 0.1)
    z0 = p.wam_get()["Z0"]
    zr = p.wam_z0_rows()
    assert z0 == zr.max()
    # explicit phi columns of every active coefficient: Z0 >= sum_z |phi(y|z)|
    tree = p.wam_tree()
    L, n = cfg["L"], cfg["nx"]
    acc = np.zeros(p.M)
    zs = [i * n + j for i in range(n >> L) for j in range(n >> L)]
    off = 0
    for lvl in range(1, L + 1):
        m = n >> lvl
        for bi in range(m):
            for bj in range(m):
                if tree[off + bi * m + bj]:
                    zs += [(m + bi) * n + bj, bi * n + m + bj, (m + bi) * n + m + bj]
        off += m * m
    for z in zs:
        rows, vals = p.phi_column(L, z)
        np.add.at(acc, rows.astype(np.int64), np.abs(vals))
    assert (acc <= z0 * (1 + 1e-12)).all()
    assert abs(acc.max() - z0) <= 1e-9 * z0


def test_fixed_point_z_majorizes():  # pin P8: mirror Z(y) in 2^-32 fixed point, terms rounded up
    cfg, p64, _, I0, d = problem_inputs("tiny", O, None)
    p = O.Problem(p64.geom, mirror=True)
    p.wam_init(d, I0, cfg["L"])
    p.wam_run(12, [4, 8], 0.1)
    zr = p.wam_z0_rows()
    assert p.wam_get()["Z0"] == zr.max()
    assert np.all(zr * 2.0**32 == np.round(zr * 2.0**32))      # exact multiples of 2^-32
    tree = p.wam_tree()
    L, n = cfg["L"], cfg["nx"]
    acc, nterm = np.zeros(p.M), np.zeros(p.M)
    zs = [i * n + j for i in range(n >> L) for j in range(n >> L)]
    off = 0
    for lvl in range(1, L + 1):
        m = n >> lvl
        for bi in range(m):
            for bj in range(m):
                if tree[off + bi * m + bj]:
                    zs += [(m + bi) * n + bj, bi * n + m + bj, (m + bi) * n + m + bj]
        off += m * m
    for z in zs:
        rows, vals = p.phi_column(L, z)
        np.add.at(acc, rows.astype(np.int64), np.abs(vals))
        np.add.at(nterm, rows.astype(np.int64), 1.0)
    # majorizes the exact sum (up to the f64 rounding of acc itself) and stays
    # within one 2^-32 per term (+1 for the approximation part) above it
    assert np.all(zr >= acc * (1 - 1e-14))
    assert np.all(zr - acc <= (nterm + 1) * 2.0**-32 + 1e-12 * acc)


def test_expand_tree_bright_block_oracle():  # SPEC.md:256, acceptance 8
    g = _geom(32, 30, 48, 1.0)
    p = O.Problem(g)
    I0 = np.full(p.M, 1e5)
    p.wam_init(p.simulate(np.zeros(p.N), I0, 0, noisy=False), I0, 3)
    # single bright 8x8 block at rows 8..15, cols 16..23 -> beta with that image
    img = np.zeros((32, 32))
    img[8:16, 16:24] = 1.0
    beta = O.dwt2(img.ravel(), 32, 32, 3)
    p.wam_init(p.simulate(np.zeros(p.N), I0, 0, noisy=False), I0, 3, init_beta=beta)
    newly = p.wam_expand(0.1)
    tree = p.wam_tree()
    lvl3 = tree[(16 * 16 + 8 * 8):]          # levels 1, 2 first, level 3 last (4x4 blocks of 8x8)
    expect = np.zeros((4, 4), np.uint8)
    expect[1, 2] = 1                          # footprint rows 8-15, cols 16-23
    assert newly == 1
    assert np.array_equal(lvl3.reshape(4, 4), expect)
    assert tree[: 16 * 16 + 8 * 8].sum() == 0
    # second event refines one level further, only under the block (closure)
    newly2 = p.wam_expand(0.1)
    lvl2 = tree2 = p.wam_tree()[16 * 16: 16 * 16 + 64].reshape(8, 8)
    assert newly2 == 4 and lvl2[2:4, 4:6].all() and tree2.sum() == 4


def test_expand_zero_image_is_noop():
    g = _geom(16, 20, 24, 2.0)
    p = O.Problem(g)
    I0 = np.full(p.M, 1e4)
    p.wam_init(p.simulate(np.zeros(p.N), I0, 0, noisy=False), I0, 2)
    assert p.wam_expand(0.1) == 0 and p.wam_tree().sum() == 0


def test_adaptivity_economy():  # acceptance 6
    cfg, p, _, I0, d = problem_inputs("tiny", O, None)
    a = O.Problem(p.geom)
    a.am_init(d, I0)
    am = a.am_iterate(100)
    target = am[-1][1]
    p.wam_init(d, I0, cfg["L"])
    recs = p.wam_run(300, [64, 128, 256], 0.1)
    assert recs[-1][3] < p.N                  # strict subset of all coefficients
    reached = [r for r in recs if r[1] <= target]
    if reached:
        assert reached[0][4] < 100 * p.N


def test_noiseless_consistency():  # acceptance 7: 32x32, RMSE < 1e-3 of range within 500 iterations
    g = _geom(32, 60, 64, 4.0)
    p = O.Problem(g)
    mu_t = O.rasterize(g, [dict(kind=1, cx=0, cy=0, cz=0, ax=40, ay=36, az=1, angle=0.0, value=0.02),
                           dict(kind=1, cx=12, cy=-8, cz=0, ax=8, ay=8, az=1, angle=0.0, value=0.05)])
    I0 = np.full(p.M, 1e5)
    d = p.simulate(mu_t, I0, 0, noisy=False)
    p.am_init(d, I0)
    p.am_iterate(500)
    rmse = np.sqrt(np.mean((p.am_get()["mu"] - mu_t) ** 2))
    assert rmse < 1e-3 * (mu_t.max() - mu_t.min())


def test_seeded_data_deterministic():
    _, p1, _, _, d1 = problem_inputs("tiny", O, None)
    _, p2, _, _, d2 = problem_inputs("tiny", O, None, threads=3)
    assert np.array_equal(d1, d2)


def test_mirror_mode_close_to_f64():  # pin P7: fp32 storage tracks f64 within 1e-4
    cfg, p64, _, I0, d = problem_inputs("tiny", O, None)
    p32 = O.Problem(p64.geom, mirror=True)
    p64.wam_init(d, I0, cfg["L"])
    p32.wam_init(d, I0, cfg["L"])
    r64 = p64.wam_run(cfg["J"], cfg["schedule"], 0.1)
    r32 = p32.wam_run(cfg["J"], cfg["schedule"], 0.1)
    o64 = np.array([r[1] for r in r64])
    o32 = np.array([r[1] for r in r32])
    assert np.linalg.norm(o64 - o32) / np.linalg.norm(o64) < 1e-4
    m64, m32 = p64.wam_get()["mu"], p32.wam_get()["mu"]
    assert np.linalg.norm(m64 - m32) / np.linalg.norm(m64) < 1e-4
    assert np.array_equal(p64.wam_tree(), p32.wam_tree())
