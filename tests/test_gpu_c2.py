"""C2 compressed CSR forward (kernels.cuh k_c2_build / k_fwd_c2): a Siddon row
is its first cell, two step signs and 2 bits per entry.  The compressed forward
uses the lane mapping and summation order of the uncompressed patch forward,
so l = H mu must be BIT-identical with C2 on (WAMGPU_C2=1, opt-in: measured
slower) and off, and the fused q / objective too."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ctx(wam, cfg, c2):
    from paper_1508_04458_b200 import configs
    old = os.environ.get("WAMGPU_C2")
    os.environ["WAMGPU_C2"] = "1" if c2 else "0"
    try:
        c = wam.Context(0)
        c.set_geometry(configs.geometry(cfg, wam.Geometry))
    finally:
        if old is None:
            os.environ.pop("WAMGPU_C2", None)
        else:
            os.environ["WAMGPU_C2"] = old
    return c


@pytest.mark.parametrize("name", ["tiny", "small", "small_lug", "cfg1"])
def test_c2_forward_bit_identical(wam, name):
    from paper_1508_04458_b200 import configs
    cfg = configs.get(name)
    a, b = _ctx(wam, cfg, True), _ctx(wam, cfg, False)
    rng = np.random.default_rng(3)
    mu = rng.uniform(0.0, 0.05, size=a.N).astype(np.float32).astype(np.float64)
    la, lb = a.forward_project(mu), b.forward_project(mu)
    assert np.array_equal(la, lb)
    # fused Beer's law + objective through an AM iteration
    from oracle import oracle as O
    og = O.make_geometry(**configs.geometry(cfg))
    p = O.Problem(og)
    mu_true = O.rasterize(og, configs.phantom(cfg))
    I0 = configs.incident(cfg, p.M)
    d = p.simulate(mu_true, I0, cfg["seed"])
    for c in (a, b):
        c.set_data(d, I0)
        c.am_init()
    ra = [r["objective"] for r in a.am_iterate(3)]
    rb = [r["objective"] for r in b.am_iterate(3)]
    assert ra == rb
    assert np.array_equal(a.image(), b.image())
    a.close(); b.close()
