"""WAMH system-matrix cache in the product (
wamrec::save/load_system_matrix, system_matrix.hpp:87-158):

* a v1 file written by the UNMODIFIED reference (oracle/_ref save_system_matrix)
  loads onto the device bit-identical (fp32 storage, pin P7) to the device's
  own build of the same matrix, CSR and CSC;
* the device's v1 file is byte-identical to the reference layout of the
  fp32-rounded matrix, and the reference's load_system_matrix reads it back;
* v2 (fp32 device layout, optional CSC mirror) round-trips byte for byte, and a
  reconstruction from a loaded v2 cache equals one from set_geometry;
* a view shard loads only its rows;
* IoError (status 4, errors.hpp:32-35) for missing, foreign, truncated and
  unsupported-version files.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_1508_04458_b200 import configs

pytestmark = pytest.mark.gpu


def _arc(name):
    cfg = configs.get(name)
    return cfg, configs.geometry(cfg)


@pytest.fixture
def tmp(tmp_path):
    return str(tmp_path)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", ["small", "cfg1"])
def test_reference_v1_file_loads_bit_exact(wam, tmp, name):
    cfg, g = _arc(name)
    og = O.make_geometry(**g)
    ref = O.RefMatrix.from_rays(cfg["nx"], cfg["ny"], cfg["voxel"], O.Problem(og).rays())
    path = os.path.join(tmp, "ref.wamh")
    ref.save(path)
    c = wam.Context(0)
    c.set_grid(cfg["nx"], cfg["ny"], 1)
    c.load_matrix_wamh(path)
    dev = wam.Context(0)
    dev.set_geometry(configs.geometry(cfg, wam.Geometry))
    rp, ci, v = ref.csr()
    a, b = c.matrix_csr(), dev.matrix_csr()
    assert np.array_equal(a[0], rp) and np.array_equal(a[1], ci) and np.array_equal(a[2], v.astype(np.float32))
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    for x, y in zip(c.matrix_csc(), dev.matrix_csc()):
        assert np.array_equal(x, y)
    # the device's v1 file: the reference layout of the fp32-rounded matrix,
    # readable by the reference's own loader
    out = os.path.join(tmp, "dev_v1.wamh")
    c.save_matrix_wamh(out, version=1)
    want = (b"WAMH" + np.uint32(1).tobytes() + np.array([ref.M, ref.N, ref.nnz], np.uint64).tobytes() +
            rp.astype(np.uint64).tobytes() + ci.astype(np.uint32).tobytes() +
            v.astype(np.float32).astype(np.float64).tobytes())
    assert open(out, "rb").read() == want
    back = O.RefMatrix.load(out)
    rp2, ci2, v2 = back.csr()
    assert np.array_equal(rp2, rp) and np.array_equal(ci2, ci) and np.array_equal(v2, v.astype(np.float32))


@pytest.mark.parametrize("with_csc", [False, True])
def test_v2_round_trip_and_reconstruction(wam, orc, tmp, with_csc):
    cfg, _ = _arc("small_lug")
    a = wam.Context(0)
    a.set_geometry(configs.geometry(cfg, wam.Geometry))
    p1 = os.path.join(tmp, "a.wamh")
    a.save_matrix_wamh(p1, version=2, with_csc=with_csc)
    size = 48 + 8 * (a.M + 1) + 8 * a.nnz + ((8 * (a.N + 1) + 8 * a.nnz) if with_csc else 0)
    assert os.path.getsize(p1) == size
    b = wam.Context(0)
    b.load_matrix_wamh(p1)                 # grid (nx, ny) travels in the v2 header
    for x, y in zip(a.matrix_csr(), b.matrix_csr()):
        assert np.array_equal(x, y)
    for x, y in zip(a.matrix_csc(), b.matrix_csc()):
        assert np.array_equal(x, y)
    p2 = os.path.join(tmp, "b.wamh")
    b.save_matrix_wamh(p2, version=2, with_csc=with_csc)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    # the same reconstruction from the cache as from the geometry
    og = orc.make_geometry(**configs.geometry(cfg))
    p = orc.Problem(og)
    I0 = configs.incident(cfg, p.M)
    d = p.simulate(orc.rasterize(og, configs.phantom(cfg)), I0, cfg["seed"])
    res = []
    for c in (a, b):
        c.set_data(d, I0)
        c.wam_init(cfg["L"])
        r = c.wam_run(cfg["J"], cfg["schedule"], 0.1)
        res.append(([x["objective"] for x in r], c.tree(), c.image()))
    assert res[0][0] == res[1][0]
    assert np.array_equal(res[0][1], res[1][1]) and np.array_equal(res[0][2], res[1][2])


def test_view_shard_loads_its_rows(wam, tmp):
    cfg, _ = _arc("small")
    full = wam.Context(0)
    full.set_geometry(configs.geometry(cfg, wam.Geometry))
    path = os.path.join(tmp, "m.wamh")
    full.save_matrix_wamh(path, version=2)
    rp, ci, v = full.matrix_csr()
    R = 3
    for k in range(R):
        c = wam.Context(0)
        c.set_comm_local(-1, k, R)
        c.load_matrix_wamh(path)
        r0, r1 = c.row0, c.row1
        srp, sci, sv = c.matrix_csr()
        lo, hi = int(rp[r0]), int(rp[r1])
        assert np.array_equal(srp, rp[r0:r1 + 1] - rp[r0])
        assert np.array_equal(sci, ci[lo:hi]) and np.array_equal(sv, v[lo:hi])
        with pytest.raises(wam.ContractError):
            c.save_matrix_wamh(os.path.join(tmp, "x.wamh"))


def test_io_errors(wam, tmp):
    c = wam.Context(0)
    with pytest.raises(wam.IoError):
        c.load_matrix_wamh(os.path.join(tmp, "missing.wamh"))
    bad = os.path.join(tmp, "bad.wamh")
    open(bad, "wb").write(b"NOPE" + bytes(60))
    with pytest.raises(wam.IoError):
        c.load_matrix_wamh(bad)
    cfg, _ = _arc("tiny")
    a = wam.Context(0)
    a.set_geometry(configs.geometry(cfg, wam.Geometry))
    good = os.path.join(tmp, "good.wamh")
    a.save_matrix_wamh(good, version=1)
    blob = open(good, "rb").read()
    open(bad, "wb").write(blob[:-5])                               # truncated
    with pytest.raises(wam.IoError):
        c.load_matrix_wamh(bad)
    open(bad, "wb").write(blob[:4] + np.uint32(3).tobytes() + blob[8:])   # unsupported version
    with pytest.raises(wam.IoError):
        c.load_matrix_wamh(bad)
    with pytest.raises(wam.IoError):
        a.save_matrix_wamh(os.path.join(tmp, "no_such_dir", "x.wamh"))
    with pytest.raises(wam.ConfigError):
        a.save_matrix_wamh(os.path.join(tmp, "x.wamh"), version=7)


def test_set_grid_after_matrix_rejected(wam):
    cfg, _ = _arc("tiny")
    a = wam.Context(0)
    a.set_geometry(configs.geometry(cfg, wam.Geometry))
    with pytest.raises(wam.ContractError):
        a.set_grid(cfg["nx"], cfg["ny"], 1)
