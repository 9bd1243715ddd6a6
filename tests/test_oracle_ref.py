"""Pins the oracle's system model bit-for-bit against the reference headers
compiled verbatim (oracle/_ref/libwamref.so, built from /root/reference by
oracle/Makefile), and the SPEC's ray-tracing examples through the reference's
own detail::trace_ray (erratum E3: validate() forbids 1x1/2x2
grids, so they go through trace_ray directly)."""
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")

GEOMS = [
    # beam, nx, ny, voxel, views, detectors, spacing
    (0, 16, 16, 1.0, 12, 24, 1.0),
    (0, 24, 16, 0.7, 30, 40, 0.61),
    (1, 32, 32, 1.0, 45, 48, 1.37),
    (1, 64, 64, 0.5, 60, 96, 0.71),
]


@pytest.mark.parametrize("beam,nx,ny,vox,V,D,sp", GEOMS)
def test_csr_csc_bit_identical_to_reference(beam, nx, ny, vox, V, D, sp):
    og = O.make_geometry(nx, ny, 1, vox, V, D, spacing=sp, beam=beam, sod=500.0, sdd=1000.0)
    p = O.Problem(og, threads=3)
    r = O.RefMatrix.build(beam, nx, ny, 1, vox, V, D, sp, 500.0, 1000.0)
    for a, b in zip(p.csr(), r.csr()):
        assert a.dtype == b.dtype and np.array_equal(a, b)
    for a, b in zip(p.csc(), r.csc()):
        assert np.array_equal(a, b)


def test_make_ray_bit_identical_to_reference():
    og = O.make_geometry(32, 32, 1, 1.0, 45, 48, spacing=1.37, beam=1)
    rays = O.Problem(og).rays()
    for v, k in [(0, 0), (3, 17), (44, 47), (22, 24)]:
        ref = O.ref_make_ray(1, 32, 32, 1.0, 45, 48, 1.37, 500.0, 1000.0, v, k)
        assert np.array_equal(rays[v * 48 + k], ref)


@pytest.mark.parametrize("name", ["tiny", "cfg1"])
def test_arc_detector_through_reference_tracer(name):
    """Pin P1: the arc rays come from the oracle, the intersection lengths from
    the unmodified reference trace_ray."""
    from paper_1508_04458_b200 import configs
    cfg = configs.get(name)
    p = O.Problem(O.make_geometry(**configs.geometry(cfg)))
    r = O.RefMatrix.from_rays(cfg["nx"], cfg["ny"], cfg["voxel"], p.rays())
    for a, b in zip(p.csr(), r.csr()):
        assert np.array_equal(a, b)
    if name == "cfg1":
        assert p.nnz == 7046648


def test_trace_ray_spec_examples():
    # 1x1 voxel, axis-aligned ray -> 1.0
    ix, iy, ln = O.ref_trace(1, 1, 1.0, [-5.0, 0.0, 1.0, 0.0, -1e300, 1e300])
    assert list(ix) == [0] and ln[0] == 1.0
    # main diagonal of a unit voxel -> sqrt(2); reference is 3 ulp off
    s = 1.0 / math.sqrt(2.0)
    ix, iy, ln = O.ref_trace(1, 1, 1.0, [-1.0, -1.0, s, s, -1e300, 1e300])
    assert len(ln) == 1 and abs(ln[0] - math.sqrt(2.0)) < 1e-15
    # 2x2 grid, horizontal ray through the lower row -> two entries of 1.0
    ix, iy, ln = O.ref_trace(2, 2, 1.0, [-5.0, -0.5, 1.0, 0.0, -1e300, 1e300])
    assert list(ix) == [0, 1] and list(iy) == [0, 0] and list(ln) == [1.0, 1.0]


def test_reference_matrix_invariants():  # SPEC.md:35-38, system_matrix.hpp:17-19
    og = O.make_geometry(32, 32, 1, 1.0, 45, 48, spacing=1.37, beam=1)
    p = O.Problem(og)
    rp, ci, v = p.csr()
    assert (v > 0).all()
    diag = math.hypot(32.0, 32.0)
    rs = np.add.reduceat(v, rp[:-1].astype(np.int64))[np.diff(rp) > 0]
    assert rs.max() <= diag
    for y in range(p.M):  # no duplicate (row, col)
        c = ci[rp[y]:rp[y + 1]]
        assert len(np.unique(c)) == len(c)
    cp, ri, _ = p.csc()
    for x in range(p.N):
        r = ri[cp[x]:cp[x + 1]]
        assert (np.diff(r.astype(np.int64)) > 0).all()


def test_wamh_cache_roundtrip(tmp_path):  # system_matrix.hpp:117-158
    R = O.reflib()
    m = O.RefMatrix.build(1, 16, 16, 1, 1.0, 10, 20, 1.2, 500.0, 1000.0)
    path = str(tmp_path / "h.wamh")
    assert R.ref_save(m.h, path.encode()) == 0
    import ctypes as C
    h = C.c_void_p()
    assert R.ref_load(path.encode(), C.byref(h)) == 0
    m2 = O.RefMatrix(h)
    assert R.ref_equal(m.h, m2.h) == 1
    assert os.path.getsize(path) == 32 + 8 * (m.M + 1) + 12 * m.nnz
