"""predicted_means / i_divergence as standalone C-ABI ops,
checked against the oracle (oracle/wam_oracle.cpp orc_predicted_means /
orc_i_divergence) and the SPEC's own worked examples.

Tolerances (fp64): exp/log on the device and in libm may differ in the last
place, and the device sum is a fixed-order tree where the oracle sums in ray
order: 1e-14 relative per mean, 1e-12 relative on the divergence."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_1508_04458_b200 as wg
    c = wg.Context(0)
    yield c
    c.close()


def test_predicted_means_spec_examples(ctx):
    # SPEC.md:86-88
    np.testing.assert_array_equal(ctx.predicted_means([3.0, 10.0], [0.0, 0.0]), [3.0, 10.0])
    q = ctx.predicted_means([10.0, 10.0], [0.5, 0.7])
    np.testing.assert_allclose(q, [6.0653066, 4.9658530], rtol=0, atol=5e-8)


def test_i_divergence_spec_examples(ctx):
    # SPEC.md:95-97
    v = np.array([0.5, 2.0, 7.0])
    assert ctx.i_divergence(v, v) == 0.0
    assert abs(ctx.i_divergence([2.0], [1.0]) - (2 * np.log(2.0) - 1.0)) < 1e-15
    assert ctx.i_divergence([0.0], [3.0]) == 3.0


@pytest.mark.parametrize("n", [1, 255, 4097, 1 << 20, 3 * (1 << 20) + 17])
def test_against_oracle(ctx, n):
    from oracle import oracle as orc
    rng = np.random.default_rng(1508 + n)
    I0 = rng.uniform(1e3, 1e5, n)
    l = rng.uniform(0.0, 6.0, n)
    q = ctx.predicted_means(I0, l)
    qo = orc.predicted_means(I0, l)
    np.testing.assert_allclose(q, qo, rtol=1e-14, atol=0)
    assert (q > 0).all()
    d = rng.poisson(qo).astype(np.float64)   # includes zero counts at the dark end
    v = ctx.i_divergence(d, qo)
    vo = orc.i_divergence(d, qo)
    assert v >= 0.0
    assert abs(v - vo) <= 1e-12 * abs(vo)
    assert ctx.i_divergence(d, qo) == v      # fixed-order sum: reproducible bit for bit


def test_empty(ctx):
    assert ctx.predicted_means(np.zeros(0), np.zeros(0)).size == 0
    assert ctx.i_divergence(np.zeros(0), np.zeros(0)) == 0.0


def test_errors(ctx):
    import paper_1508_04458_b200 as wg
    l = np.zeros(5000)
    l[4321] = np.inf
    l[4800] = np.nan
    with pytest.raises(wg.NumericError, match="ray 4321"):
        ctx.predicted_means(np.ones(5000), l)
    q = np.ones(5000)
    q[77] = 0.0
    q[4000] = -1.0
    with pytest.raises(wg.NumericError, match="ray 77"):
        ctx.i_divergence(np.ones(5000), q)
    with pytest.raises(wg.ContractError):
        ctx.predicted_means(np.ones(3), np.ones(4))
    with pytest.raises(wg.ContractError):
        ctx.i_divergence(np.ones(3), np.ones(4))
