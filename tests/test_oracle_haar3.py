"""Separable 3D Haar (pin P3) in the oracle: transform
properties, the factorised phi(y_s|z) = psi(y|b) c^l sigma_z(s) checked against
brute-force columns H (Omega_3 e_z), Z0 validity, monotone I-divergence and
mirror-vs-f64 agreement (tree identical)."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from wam_testutil import problem_inputs


def test_dwt3_parseval_pr_constant():
    rng = np.random.default_rng(4)
    for (nx, ny, nz, L) in [(16, 16, 8, 3), (8, 16, 4, 2), (32, 32, 16, 4)]:
        x = rng.standard_normal(nx * ny * nz)
        y = O.dwt3(x, nx, ny, nz, L)
        assert abs(np.linalg.norm(y) - np.linalg.norm(x)) <= 1e-12 * np.linalg.norm(x)
        assert np.abs(O.idwt3(y, nx, ny, nz, L) - x).max() < 1e-12
        c = O.dwt3(np.full(nx * ny * nz, 0.7), nx, ny, nz, L).reshape(nz, ny, nx)
        a = c[: nz >> L, : ny >> L, : nx >> L]
        assert np.allclose(a, 0.7 * 2 ** (1.5 * L), rtol=1e-12)
        c[: nz >> L, : ny >> L, : nx >> L] = 0
        assert np.abs(c).max() < 1e-12
    with pytest.raises(O.OracleError) as e:
        O.dwt3(np.zeros(16 * 16 * 6), 16, 16, 6, 2)
    assert e.value.code == 1


def _small3d():
    g = O.make_geometry(16, 16, 4, 4.0, 20, 24, beam=2, dgamma=2 * math.asin(32.0 / 500.0) / 24)
    return g


def test_z_rows_match_brute_force_columns():
    g = _small3d()
    p = O.Problem(g)
    p.set_haar_dim(3)
    I0 = np.full(p.M * p.nz, 1e5)
    mu_t = O.rasterize(g, [dict(kind=0, cx=2, cy=-3, cz=1, ax=20, ay=14, az=6, angle=0.3, value=0.04),
                           dict(kind=1, cx=-8, cy=6, cz=-2, ax=4, ay=4, az=3, angle=0.0, value=0.6)])
    d = p.simulate(mu_t, I0, 3)
    L = 2
    p.wam_init(d, I0, L)
    p.wam_iterate(3)
    p.wam_expand(0.1)
    p.wam_iterate(2)
    p.wam_expand(0.1)
    tree = p.wam_tree()
    nx, ny, nz, N = 16, 16, 4, 256
    # active coefficients (3D Mallat), brute-force columns phi(.|z) = H(Omega_3 e_z) per slice
    act = []
    for k in range(nz >> L):
        for bi in range(ny >> L):
            for bj in range(nx >> L):
                act.append(k * N + bi * nx + bj)
    off = 0
    for l in range(1, L + 1):
        dl, hl, wl = nz >> l, ny >> l, nx >> l
        for k in range(dl):
            for bi in range(hl):
                for bj in range(wl):
                    if tree[off + (k * hl + bi) * wl + bj]:
                        for (zz, yy, xx) in [(k, hl + bi, bj), (k, bi, wl + bj), (k, hl + bi, wl + bj),
                                             (dl + k, bi, bj), (dl + k, hl + bi, bj), (dl + k, bi, wl + bj),
                                             (dl + k, hl + bi, wl + bj)]:
                            act.append(zz * N + yy * nx + xx)
        off += dl * hl * wl
    Z = np.zeros(p.M * nz)
    for z in act:
        e = np.zeros(N * nz)
        e[z] = 1.0
        col = p.forward_project(O.idwt3(e, nx, ny, nz, L))
        Z += np.abs(col)
    Zys = Z.reshape(nz, p.M)
    zr = p.wam_z0_rows()
    assert np.allclose(zr, Zys.max(axis=0), rtol=1e-10, atol=1e-12)
    assert p.wam_get()["Z0"] == zr.max()


@pytest.mark.parametrize("mirror", [0, 1])
def test_wam3d_monotone(mirror):
    cfg, p, _, I0, d = problem_inputs("tiny3d", O, None, mirror=mirror)
    p.set_haar_dim(3)
    p.wam_init(d, I0, cfg["L"])
    recs = p.wam_run(cfg["J"], cfg["schedule"], 0.1)
    obj = [r[1] for r in recs]
    assert all(b <= a * (1 + 1e-9) for a, b in zip(obj, obj[1:]))
    assert recs[-1][3] > recs[0][3]


def test_wam3d_mirror_close_to_f64():
    cfg, p64, _, I0, d = problem_inputs("tiny3d", O, None)
    p32 = O.Problem(p64.geom, mirror=True)
    for p in (p64, p32):
        p.set_haar_dim(3)
        p.wam_init(d, I0, cfg["L"])
    r64 = p64.wam_run(cfg["J"], cfg["schedule"], 0.1)
    r32 = p32.wam_run(cfg["J"], cfg["schedule"], 0.1)
    o64, o32 = np.array([r[1] for r in r64]), np.array([r[1] for r in r32])
    assert np.linalg.norm(o64 - o32) / np.linalg.norm(o64) < 1e-4
    assert np.array_equal(p64.wam_tree(), p32.wam_tree())
    m64, m32 = p64.wam_get()["mu"], p32.wam_get()["mu"]
    assert np.linalg.norm(m64 - m32) / np.linalg.norm(m64) < 1e-4
