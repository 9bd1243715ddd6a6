"""Seeded simulation on the device (simulate_counts
SPEC.md:153-161): wamgpu_simulate_device restates the host simulator
(host_model.cpp simulate) operation for operation, so the Poisson counts are
identical to the host's -- and to the oracle's, which the golden fixtures pin
(tests/test_golden.py).  Noiseless means may differ by the last bits of exp."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["tiny", "tiny3d", "small3d", "cfg1"])
def test_device_simulation_equals_host(wam, name):
    from paper_1508_04458_b200 import configs
    cfg = configs.get(name)
    g = configs.geometry(cfg, wam.Geometry)
    mu = wam.rasterize(g, configs.phantom(cfg))
    I0 = configs.incident(cfg, cfg["views"] * cfg["detectors"])
    d_host = wam.simulate(g, mu, I0, cfg["seed"])
    d_dev = wam.simulate_device(g, mu, I0, cfg["seed"])
    assert np.array_equal(d_dev, d_host)
    m_host = wam.simulate(g, mu, I0, cfg["seed"], noisy=False)
    m_dev = wam.simulate_device(g, mu, I0, cfg["seed"], noisy=False)
    assert np.max(np.abs(m_dev - m_host) / np.maximum(m_host, 1e-300)) <= 4e-16


def test_device_simulation_rejects_bad_means(wam):
    from paper_1508_04458_b200 import configs
    cfg = configs.get("tiny")
    g = configs.geometry(cfg, wam.Geometry)
    mu = wam.rasterize(g, configs.phantom(cfg))
    I0 = configs.incident(cfg, cfg["views"] * cfg["detectors"])
    I0[5] = np.inf
    with pytest.raises(wam.NumericError):
        wam.simulate_device(g, mu, I0, cfg["seed"])
