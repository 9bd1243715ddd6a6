"""The oracle's scalable modes used for the BASELINE-size goldens
(tests/golden/make_golden_big.py) give bit-identical results to the plain
problem:

* slim (CSR only, no exact-h copy, no CSC; fp32 h in mirror mode): back
  projection becomes an ascending-ray CSR scatter, which adds every voxel's terms
  in the CSC order;
* the slab (voxel-major) 3D loops and the block-driven 3D splits keep each
  sum's order;
* the reference-precision splits no longer depend on the thread count (fixed
  ray chunks in 2D, one ordered chain per coefficient in 3D).
"""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1508_04458_b200 import configs


def _run(name, mirror, slim, algo, threads=0):
    cfg = configs.get(name)
    og = O.make_geometry(**configs.geometry(cfg))
    p = O.Problem(og, mirror=mirror, slim=slim, threads=threads)
    mu = O.rasterize(og, configs.phantom(cfg))
    I0 = configs.incident(cfg, p.M)
    d = p.simulate(mu, I0, cfg["seed"])
    if algo == "am":
        p.am_init(d, I0)
        r = [x[1] for x in p.am_iterate(3)]
        return d, r, p.am_get()["mu"]
    if cfg["nz"] > 1:
        p.set_haar_dim(cfg["haar"] if cfg["haar"] == 3 else 3)
    p.wam_init(d, I0, cfg["L"])
    r = [x[1] for x in p.wam_run(cfg["J"], cfg["schedule"])]
    return d, r, p.wam_get()["beta"], p.wam_tree(), p.wam_get()["Z0"]


@pytest.mark.parametrize("name", ["tiny3d", "tiny3d64"])
@pytest.mark.parametrize("mirror", [False, True])
@pytest.mark.parametrize("algo", ["am", "wam"])
def test_slim_problem_bit_identical(name, mirror, algo):
    a = _run(name, mirror, False, algo)
    b = _run(name, mirror, True, algo)
    for x, y in zip(a, b):
        assert np.array_equal(np.asarray(x), np.asarray(y))


def test_slim_has_no_csc():
    cfg = configs.get("tiny3d")
    p = O.Problem(O.make_geometry(**configs.geometry(cfg)), slim=True)
    with pytest.raises(O.OracleError):
        p.csc()


@pytest.mark.parametrize("name", ["tiny", "tiny3d"])
def test_reference_precision_split_independent_of_threads(name):
    a = _run(name, False, False, "wam", threads=1)
    b = _run(name, False, False, "wam", threads=5)
    for x, y in zip(a, b):
        assert np.array_equal(np.asarray(x), np.asarray(y))
