"""Known-answer tests of the CPU oracle against the SPEC's examples,
with errata E1-E3 of SURVEY.md App. A applied.  Pins the oracle before it is
trusted as the GPU's checker."""
import math

import numpy as np
import pytest

from oracle import oracle as O


def test_beer_law_examples():
    q = O.predicted_means([10.0, 10.0, 7.0], [0.5, 0.7, 0.0])
    assert abs(q[0] - 6.0653066) < 1e-7
    assert abs(q[1] - 4.9658530) < 1e-7
    assert q[2] == 7.0


def test_beer_law_nonfinite_is_numeric_error():
    with pytest.raises(O.OracleError) as e:
        O.predicted_means([1.0], [float("nan")])
    assert e.value.code == 3


def test_i_divergence_examples():
    assert abs(O.i_divergence([2.0], [1.0]) - (2 * math.log(2) - 1)) < 1e-15
    assert abs(O.i_divergence([2.0], [1.0]) - 0.3862944) < 1e-7
    assert O.i_divergence([0.0], [3.0]) == 3.0
    q = np.array([1.5, 2.0, 7.25])
    assert O.i_divergence(q, q) == 0.0
    with pytest.raises(O.OracleError) as e:
        O.i_divergence([1.0], [0.0])
    assert e.value.code == 3


def test_forward_back_hand_examples():  # H = [[1,0],[1,1]]
    p = O.Problem.from_csr([0, 1, 3], [0, 0, 1], [1.0, 1.0, 1.0], nx=2, ny=1)
    assert np.allclose(p.forward_project([0.5, 0.2]), [0.5, 0.7], rtol=0, atol=1e-15)
    assert np.array_equal(p.back_project([1.0, 2.0]), [3.0, 2.0])
    assert np.array_equal(p.forward_project([0.0, 0.0]), [0.0, 0.0])
    assert np.array_equal(p.back_project([0.0, 0.0]), [0.0, 0.0])
    mu = np.array([0.3, 0.9])
    assert np.allclose(p.forward_project(3 * mu), 3 * p.forward_project(mu), rtol=1e-15)


def test_am_scalar_example():  # 1 voxel, 1 ray, h=1, I0=10, d=5
    p = O.Problem.from_csr([0, 1], [0], [1.0], nx=1, ny=1)
    p.am_init([5.0], [10.0])
    st = p.am_get()
    assert st["Z0"] == 1.0 and st["b"][0] == 5.0
    recs = p.am_iterate(1)
    st = p.am_get()
    assert abs(st["mu"][0] - math.log(2.0)) < 1e-15
    assert abs(st["q"][0] - 5.0) < 1e-12
    assert abs(recs[0][1]) < 1e-12            # I(d||q) = 0 at the fixed point
    p.am_iterate(1)
    assert abs(p.am_get()["mu"][0] - math.log(2.0)) < 1e-12


def test_am_zero_phantom_fixed_point():
    g = O.make_geometry(8, 8, 1, 1.0, 12, 16, beam=2, dgamma=0.01)
    p = O.Problem(g)
    I0 = np.full(p.M, 100.0)
    d = p.simulate(np.zeros(p.N), I0, 0, noisy=False)
    assert np.array_equal(d, I0)
    p.am_init(d, I0)
    p.am_iterate(3)
    assert np.array_equal(p.am_get()["mu"], np.zeros(p.N))


def test_root_solver_examples():  # SPEC.md:368-370 with erratum E1
    r, v = O.solve_update(2.0, 3.0, -1.0, 1.0, 0.0)
    assert r == 0 and abs(v) < 1e-15                 # u = 1, no change
    r, v = O.solve_update(5.0, 10.0, 0.0, 1.0, 0.0)
    assert r == 0 and abs(v - math.log(2.0)) < 1e-15  # E2: u = b / b+
    r, v = O.solve_update(2.0, 4.0, -1.0, 1.0, 0.0)
    u = (1 + math.sqrt(5)) / 4
    assert abs(math.exp(-v) - u) < 1e-15
    assert abs(v - 0.21193536) < 1e-8                # E1: SPEC prints 0.212230 (wrong)
    assert abs(v - 0.212230) > 1e-4


def test_root_solver_degenerate_cases():
    assert O.solve_update(1.0, 0.0, 0.0, 1.0, 0.5) == (1, 0.5)       # skipped
    assert O.solve_update(-1.0, 2.0, 0.0, 1.0, 0.5) == (2, 0.5)      # b<=0, b-=0
    assert O.solve_update(1.0, 0.0, -2.0, 1.0, 0.5) == (2, 0.5)      # b+=0, b>=0
    r, v = O.solve_update(-1.0, 0.0, -2.0, 2.0, 0.5)                 # b+=0, b<0: u = b-/b
    assert r == 0 and abs(v - (0.5 - math.log(2.0) / 2.0)) < 1e-15


def test_root_solver_vs_bisection():  # acceptance 3: 1000 tuples
    rng = np.random.default_rng(1234)
    for _ in range(1000):
        bp = float(rng.uniform(0.01, 100))
        bm = -float(rng.uniform(0.0, 50)) if rng.random() < 0.7 else 0.0
        b = float(rng.uniform(0.01, 120)) if bm == 0.0 else float(rng.uniform(-60, 120))
        Z0 = float(rng.uniform(0.5, 50))
        beta = float(rng.uniform(-1, 1))
        r, v = O.solve_update(b, bp, bm, Z0, beta)
        assert r == 0
        grad = lambda t: b - bp * math.exp(-Z0 * (t - beta)) - bm * math.exp(Z0 * (t - beta))  # noqa: E731
        assert abs(grad(v)) <= 1e-10 * (bp - bm + abs(b))
        # bisection on u = exp(-Z0 (t - beta)): f(u) = bp u^2 - b u + bm, increasing for u > u*
        lo, hi = 1e-300, 1.0
        f = lambda u: bp * u * u - b * u + bm  # noqa: E731
        while f(hi) < 0:
            hi *= 2
        for _ in range(400):
            mid = 0.5 * (lo + hi)
            if f(mid) < 0:
                lo = mid
            else:
                hi = mid
        u = math.exp(-Z0 * (v - beta))
        assert abs(u - 0.5 * (lo + hi)) <= 1e-12 * max(1.0, u)


def test_haar_examples():
    a, b, c, d = 1.0, 2.0, 3.0, 5.0
    x = np.array([a, b, c, d])
    y = O.dwt2(x, 2, 2, 1)
    H = 0.5 * np.array([[1, 1, 1, 1], [1, 1, -1, -1], [1, -1, 1, -1], [1, -1, -1, 1]])
    # Mallat positions: (0,0)=A, (1,0)=H, (0,1)=V, (1,1)=D -> flat [A, V, H, D]
    ref = H @ x
    assert np.allclose(y, [ref[0], ref[2], ref[1], ref[3]], atol=1e-15)
    for L in (1, 2, 3):
        cst = np.full(64, 0.7)
        t = O.dwt2(cst, 8, 8, L)
        n = 8 >> L
        A = t.reshape(8, 8)[:n, :n]
        assert np.allclose(A, 0.7 * 2 ** L, rtol=1e-15)
        det = t.reshape(8, 8).copy()
        det[:n, :n] = 0
        assert np.abs(det).max() == 0.0
    z = np.zeros(4)
    z[0] = 1.0
    assert np.allclose(O.idwt2(z, 2, 2, 1), 0.5)           # single approx coefficient -> block of 1/2
    assert np.array_equal(O.idwt2(np.zeros(16), 4, 4, 2), np.zeros(16))


def test_haar_pr_parseval_random():  # SPEC.md:220, 227, acceptance 4
    rng = np.random.default_rng(7)
    for _ in range(100):
        x = rng.standard_normal(32 * 32)
        y = O.dwt2(x, 32, 32, 3)
        assert abs(np.linalg.norm(y) - np.linalg.norm(x)) <= 1e-12 * np.linalg.norm(x)
        assert np.abs(O.idwt2(y, 32, 32, 3) - x).max() < 1e-12


def test_haar_indivisible_is_config_error():  # SPEC.md:214, erratum E4
    with pytest.raises(O.OracleError) as e:
        O.dwt2(np.zeros(12 * 12), 12, 12, 3)
    assert e.value.code == 1


def test_init_state_active_count():  # 32x32, L=3 -> 16 approx coefficients
    g = O.make_geometry(32, 32, 1, 1.0, 20, 32, beam=2, dgamma=0.01)
    p = O.Problem(g)
    I0 = np.full(p.M, 1e4)
    d = p.simulate(np.zeros(p.N), I0, 1, noisy=False)
    p.wam_init(d, I0, 3)
    assert p.wam_counters()["active_set"] == 16
    assert np.array_equal(p.wam_get()["q"], I0)               # init_beta = 0 -> q = I0


def test_phi_column_hand_example():  # two vertical rays, level-1 approx -> [1, 1]
    # 2x2 slice, H = [[1,0,1,0],[0,1,0,1]]
    p = O.Problem.from_csr([0, 2, 4], [0, 2, 1, 3], [1.0, 1.0, 1.0, 1.0], nx=2, ny=2)
    rows, vals = p.phi_column(1, 0)
    assert list(rows) == [0, 1] and np.allclose(vals, [1.0, 1.0])
    # identity special case L = 0: phi(.|z) is the z-th column of H
    rows, vals = p.phi_column(0, 2)
    assert list(rows) == [0] and vals[0] == 1.0


def test_rasterize_examples():
    g = O.make_geometry(32, 32, 1, 1.0, 4, 8, beam=2, dgamma=0.01)
    assert np.array_equal(O.rasterize(g, []), np.zeros(32 * 32))
    full = [dict(kind=1, cx=0, cy=0, cz=0, ax=100, ay=100, az=1, angle=0, value=0.2)]
    assert np.array_equal(O.rasterize(g, full), np.full(32 * 32, 0.2))
    disk = [dict(kind=0, cx=0, cy=0, cz=0, ax=10, ay=10, az=1, angle=0, value=0.4)]
    n = int((O.rasterize(g, disk) > 0).sum())
    assert abs(n - math.pi * 100) <= 4


def test_poisson_sampler():
    m = 1e4 * math.exp(-0.5)
    xs = np.array([O.poisson(99, k, m) for k in range(10000)])
    assert abs(xs.mean() - m) < 3 * math.sqrt(m / xs.size)
    assert abs(xs.var() / m - 1.0) < 0.05
    small = np.array([O.poisson(5, k, 3.0) for k in range(20000)])
    assert abs(small.mean() - 3.0) < 3 * math.sqrt(3.0 / small.size)
    assert O.poisson(5, 1, 7.5) == O.poisson(5, 1, 7.5)  # seeded determinism
