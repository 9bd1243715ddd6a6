"""Block-coarsened projections of the 3D wavelet-AM iteration (kernels3c.cuh):
while the finest active tree level is lf > 1, forward and back projection run
over the 2^(lf-1)-coarsened matrices (and, mode 2, on z-groups of 2^(lf-1) slices).  The run must equal the pixel-path run
(WAMGPU_COARSE=0): identical trees and counters, objectives and images within
the association error of fp64 sums; WAMGPU_COARSE_CHECK verifies on the device
that mu is constant on the blocks before every coarse forward.  Parity against
the oracle is covered by tests/test_gpu_parity3d.py, which runs with the
coarse path on (the default)."""
import os

import numpy as np
import pytest

from wam_testutil import problem_inputs, rel_l2

pytestmark = pytest.mark.gpu


def _run(W, cfg, I0, d, coarse, coarse_update=1, stats=False):
    from paper_1508_04458_b200 import configs
    os.environ["WAMGPU_COARSE"] = str(int(coarse))
    os.environ["WAMGPU_COARSE_UPDATE"] = str(int(coarse_update))
    os.environ["WAMGPU_COARSE_CHECK"] = "1"
    try:
        c = W.Context(0)
        c.set_geometry(configs.geometry(cfg, W.Geometry))
        if cfg["nz"] > 1:
            c.set_haar_dim(3)
        c.set_data(d, I0)
        c.wam_init(cfg["L"])
        obj, trees, done, st = [], [], 0, []
        for ev in cfg["schedule"] + [cfg["J"]]:
            obj += [r["objective"] for r in c.wam_iterate(ev - done)]
            done = ev
            if stats:
                st.append([a.copy() for a in c.stats()])
            if ev == cfg["J"]:
                break
            c.wam_expand(0.1)
            trees.append(c.tree().copy())
        out = dict(obj=np.array(obj), trees=trees, mu=c.image(), beta=c.beta(), scal=c.scalars(), stats=st,
                   launches=c.timing()["kernel_launches"])
        c.close()
        return out
    finally:
        os.environ.pop("WAMGPU_COARSE", None)
        os.environ.pop("WAMGPU_COARSE_UPDATE", None)
        os.environ.pop("WAMGPU_COARSE_CHECK", None)


@pytest.mark.parametrize("mode", [1, 2])   # 1: in-plane blocks; 2 (default): in-plane blocks and z-groups
@pytest.mark.parametrize("name", ["tiny3d16", "tiny3d64", "small3d"])
def test_coarse_projections_equal_the_pixel_path(wam, orc, name, mode):
    cfg, _, _, I0, d = problem_inputs(name, orc, wam)
    a = _run(wam, cfg, I0, d, coarse=mode)
    b = _run(wam, cfg, I0, d, coarse=0)
    assert len(a["trees"]) == len(b["trees"]) > 0
    for ta, tb in zip(a["trees"], b["trees"]):
        assert np.array_equal(ta, tb)
    assert a["scal"] == b["scal"]
    assert rel_l2(a["obj"], b["obj"]) < 1e-12
    assert rel_l2(a["mu"], b["mu"]) < 1e-6 and rel_l2(a["beta"], b["beta"]) < 1e-6


@pytest.mark.parametrize("name", ["tiny", "small", "small_lug", "cfg1"])
def test_coarse_projections_2d(wam, orc, name):
    """2D wavelet AM: the CSR patch forward and the CSC back projection over Hc."""
    cfg, _, _, I0, d = problem_inputs(name, orc, wam)
    a = _run(wam, cfg, I0, d, coarse=2)
    b = _run(wam, cfg, I0, d, coarse=0)
    assert len(a["trees"]) == len(b["trees"]) > 0
    for ta, tb in zip(a["trees"], b["trees"]):
        assert np.array_equal(ta, tb)
    assert a["scal"] == b["scal"]
    assert rel_l2(a["obj"], b["obj"]) < 1e-12
    assert rel_l2(a["mu"], b["mu"]) < 1e-6 and rel_l2(a["beta"], b["beta"]) < 1e-6


@pytest.mark.parametrize("name", ["tiny3d16", "tiny3d64", "small3d"])
def test_coarse_domain_update_is_bit_identical(wam, orc, name):
    """k_tile3hc (update on the (TS >> k)^3 corner of every tile, fed by the cube
    sums of g) against the full-tile update after expanding g to voxels: the same
    roundings in the same order, so objectives, beta, mu, trees and counters are
    EQUAL; b+ / b- read between phases (k_tile3h mode 3 on demand) too."""
    cfg, _, _, I0, d = problem_inputs(name, orc, wam)
    a = _run(wam, cfg, I0, d, coarse=2, coarse_update=1, stats=True)
    b = _run(wam, cfg, I0, d, coarse=2, coarse_update=0, stats=True)
    assert np.array_equal(a["obj"], b["obj"])
    assert np.array_equal(a["beta"], b["beta"]) and np.array_equal(a["mu"], b["mu"])
    assert a["scal"] == b["scal"] and all(np.array_equal(x, y) for x, y in zip(a["trees"], b["trees"]))
    assert len(a["stats"]) == len(b["stats"]) > 1
    for sa, sb in zip(a["stats"], b["stats"]):
        for x, y in zip(sa, sb):
            assert np.array_equal(x, y)
