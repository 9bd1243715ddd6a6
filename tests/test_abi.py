"""CPU-side checks of the C-ABI boundary: libwamgpu.so builds, loads, and exports
every entry point include/wamgpu.h declares; the Python mirror's host logic
(configs, schedules, error mapping) behaves; the product's host-side phantom
simulator and ray table are bit-identical to the oracle's."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "wamgpu.h")).read()
    return sorted(set(re.findall(r"\b(wamgpu_[a-z0-9_]+)\s*\(", src)))


def test_header_matches_python_mirror(wam):
    assert _declared() == sorted(wam.EXPORTED)


def test_library_exports_every_symbol(wam):
    lib = wam.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.wamgpu_version() == 1


def test_create_without_gpu_fails_loudly(wam):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    with pytest.raises(wam.CudaError):
        wam.Context(0)


def test_no_oracle_in_product():
    pkg = os.path.join(ROOT, "paper_1508_04458_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liborc" not in txt and "wam_oracle" not in txt, f


def test_schedule_pin():  # pin P4
    from paper_1508_04458_b200 import configs
    assert configs.get("cfg1")["schedule"] == [5, 10, 15]
    assert configs.get("cfg2")["schedule"] == [10, 20, 30, 40]
    assert configs.get("cfg3")["schedule"] == [7, 15, 22]
    assert configs.get("cfg4")["schedule"] == [8, 16, 24, 32]


def test_phantom_ranges():
    from paper_1508_04458_b200 import configs
    p = configs.phantom(configs.get("cfg2"))
    metal = [q for q in p if q["value"] >= 0.5]
    soft = [q for q in p[1:] if q["value"] < 0.5]
    assert 4 <= len(metal) <= 8 and all(q["value"] <= 1.5 for q in metal)
    assert 30 <= len(soft) <= 60 and all(0 <= q["value"] <= 0.06 for q in soft)
    b = configs.phantom(configs.get("cfg1"))
    assert b[0]["value"] == 0.02 and sum(q["value"] == 0.5 for q in b) == 2
    assert 6 <= sum(0.005 <= q["value"] <= 0.05 for q in b[1:]) <= 10


def test_cfg4_gain_pin():  # P6
    from paper_1508_04458_b200 import configs
    cfg = configs.get("cfg4")
    I0 = configs.incident(dict(cfg, nz=1, views=2), 2 * cfg["detectors"])
    g = I0[: cfg["detectors"]] / 1e5
    assert g.min() >= 0.8 and g.max() <= 1.2 and np.array_equal(I0[:1024], I0[1024:])


@pytest.mark.parametrize("name", ["tiny", "cfg1"])
def test_host_simulator_and_rays_match_oracle(wam, orc, name):
    from paper_1508_04458_b200 import configs
    cfg = configs.get(name)
    g = configs.geometry(cfg, wam.Geometry)
    og = orc.make_geometry(**configs.geometry(cfg))
    prims = configs.phantom(cfg)
    mu = wam.rasterize(g, prims)
    assert np.array_equal(mu, orc.rasterize(og, prims))
    p = orc.Problem(og)
    assert np.array_equal(wam.host_rays(g), p.rays())
    I0 = configs.incident(cfg, p.M)
    assert np.array_equal(wam.simulate(g, mu, I0, cfg["seed"]), p.simulate(mu, I0, cfg["seed"]))


def test_host_validation_maps_to_config_error(wam):
    g = wam.make_fan_geometry(2, 2, 1, 1.0, 10, 10, 1.0, 500.0, 1000.0)
    with pytest.raises(wam.ConfigError):
        wam.host_rays(g)
    g = wam.make_fan_geometry(8, 8, 1, 1.0, 10, 10, 1.0, 500.0, 400.0)
    with pytest.raises(wam.ConfigError):
        wam.host_rays(g)
