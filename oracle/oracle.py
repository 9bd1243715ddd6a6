"""ctypes binding of the CPU oracle (liborc.so) and of the reference shim
(oracle/_ref/libwamref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package
(paper_1508_04458_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# ORC_LIB: an alternative build of the same source (bench.py's CPU legs build
# one with -march=native on the host they time; -ffp-contract=off keeps it
# bit-identical)
_LIB = os.environ.get("ORC_LIB") or os.path.join(HERE, "liborc.so")
_REFLIB = os.path.join(HERE, "_ref", "libwamref.so")

_d = C.POINTER(C.c_double)
_u64 = C.POINTER(C.c_uint64)
_u32 = C.POINTER(C.c_uint32)
_i64 = C.POINTER(C.c_int64)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Geometry(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("voxel_size", C.c_double),
                ("detectors", C.c_int), ("detector_spacing", C.c_double), ("views", C.c_int),
                ("view_angles", _d), ("beam", C.c_int), ("source_to_center", C.c_double),
                ("source_to_detector", C.c_double), ("fan_angle_step", C.c_double)]


class Primitive(C.Structure):
    _fields_ = [("kind", C.c_int)] + [(n, C.c_double) for n in
                                      ("cx", "cy", "cz", "ax", "ay", "az", "angle", "value")]


class Record(C.Structure):
    _fields_ = [("iter", C.c_int), ("objective", C.c_double), ("elapsed_s", C.c_double),
                ("active_set", C.c_int64), ("cum_updates", C.c_int64)]


def build():
    """Compile liborc.so (and oracle/_ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def build_native(out_dir):
    """liborc.so tuned for THIS host (-march=native; -ffp-contract=off keeps
    every result bit-identical to the portable build).  Returns its path, or
    None when no compiler is available."""
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, "liborc.so")
    cmd = ["g++", "-std=c++20", "-O3", "-march=native", "-ffp-contract=off", "-fPIC", "-pthread", "-shared",
           "-o", out, os.path.join(HERE, "wam_oracle.cpp")]
    try:
        subprocess.run(cmd, check=True, capture_output=True)
    except Exception:
        return None
    return out


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        _lib = C.CDLL(_LIB)
        _lib.orc_last_error.restype = C.c_char_p
        _lib.orc_uniform.restype = C.c_double
        _lib.orc_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        _lib.orc_poisson.restype = C.c_double
        _lib.orc_poisson.argtypes = [C.c_uint64, C.c_uint64, C.c_double]
        _lib.orc_solve_update.argtypes = [C.c_double] * 5 + [_d]
        _lib.orc_create.argtypes = [C.POINTER(Geometry), C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        _lib.orc_create_ex.argtypes = [C.POINTER(Geometry), C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        _lib.orc_destroy.argtypes = [C.c_void_p]
        _lib.orc_destroy.restype = None
    return _lib


def ref_available():
    return os.path.exists(_REFLIB)


def reflib():
    global _ref
    if _ref is None:
        _ref = C.CDLL(_REFLIB)
        _ref.ref_last_error.restype = C.c_char_p
        _ref.ref_row_sum.restype = C.c_double
        _ref.ref_row_sum.argtypes = [C.c_void_p, C.c_uint64]
    return _ref


def _chk(rc, L=None):
    if rc != 0:
        L = L or lib()
        fn = L.orc_last_error if hasattr(L, "orc_last_error") else L.ref_last_error
        raise OracleError(rc, fn().decode())


def P(a, ct=C.c_double):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


def make_geometry(nx, ny, nz, voxel, views, detectors, spacing=1.0, beam=2, sod=500.0, sdd=1000.0,
                  dgamma=0.0, angles=None):
    g = Geometry(nx, ny, nz, voxel, detectors, spacing, views, None, beam, sod, sdd, dgamma)
    keep = None
    if angles is not None:
        keep = np.ascontiguousarray(angles, dtype=np.float64)
        g.view_angles = P(keep)
    g._keep = keep
    return g


class Problem:
    """Oracle problem: geometry + system matrix + AM/WAM state (f64 or fp32-mirror)."""

    def __init__(self, geom: Geometry, mirror=False, threads=0, slim=False):
        """slim: CSR only (no exact-h copy, no CSC mirror; fp32 h in mirror mode),
        bit-identical results; the memory mode for cfg4."""
        L = lib()
        h = C.c_void_p()
        _chk(L.orc_create_ex(C.byref(geom), int(mirror), int(threads), 1 if slim else 0, C.byref(h)))
        self.h = h
        self.geom = geom
        M, N, nnz, nz = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_int()
        _chk(L.orc_dims(h, C.byref(M), C.byref(N), C.byref(nnz), C.byref(nz)))
        self.M, self.N, self.nnz, self.nz = M.value, N.value, nnz.value, nz.value
        self.L = None

    @classmethod
    def from_csr(cls, row_ptr, col, val, nx, ny, mirror=False, threads=1):
        L = lib()
        self = cls.__new__(cls)
        rp = np.ascontiguousarray(row_ptr, np.uint64)
        ci = np.ascontiguousarray(col, np.uint32)
        v = np.ascontiguousarray(val, np.float64)
        h = C.c_void_p()
        _chk(L.orc_create_csr(C.c_uint64(rp.size - 1), int(nx), int(ny), P(rp, C.c_uint64), P(ci, C.c_uint32),
                              P(v), int(mirror), int(threads), C.byref(h)))
        self.h = h
        self.geom = None
        M, N, nnz, nz = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_int()
        _chk(L.orc_dims(h, C.byref(M), C.byref(N), C.byref(nnz), C.byref(nz)))
        self.M, self.N, self.nnz, self.nz = M.value, N.value, nnz.value, nz.value
        self.L = None
        return self

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_destroy(self.h)
            self.h = None

    def am_set_clamp(self, clamp):
        _chk(lib().orc_am_set_clamp(self.h, int(clamp)))

    # --- matrix
    def csr(self):
        rp = np.empty(self.M + 1, np.uint64)
        ci = np.empty(self.nnz, np.uint32)
        v = np.empty(self.nnz, np.float64)
        _chk(lib().orc_get_csr(self.h, P(rp, C.c_uint64), P(ci, C.c_uint32), P(v)))
        return rp, ci, v

    def csc(self):
        cp = np.empty(self.N + 1, np.uint64)
        ri = np.empty(self.nnz, np.uint32)
        v = np.empty(self.nnz, np.float64)
        _chk(lib().orc_get_csc(self.h, P(cp, C.c_uint64), P(ri, C.c_uint32), P(v)))
        return cp, ri, v

    def rays(self):
        r = np.empty((self.M, 6), np.float64)
        _chk(lib().orc_get_rays(self.h, P(r)))
        return r

    # --- core-model
    def forward_project(self, mu):
        mu = np.ascontiguousarray(mu, np.float64)
        out = np.empty(self.M * self.nz)
        _chk(lib().orc_forward_project(self.h, P(mu), P(out)))
        return out

    def back_project(self, w):
        w = np.ascontiguousarray(w, np.float64)
        out = np.empty(self.N * self.nz)
        _chk(lib().orc_back_project(self.h, P(w), P(out)))
        return out

    def simulate(self, mu_true, I0, seed, noisy=True):
        mu_true = np.ascontiguousarray(mu_true, np.float64)
        I0 = np.ascontiguousarray(I0, np.float64)
        d = np.empty(self.M * self.nz)
        _chk(lib().orc_simulate(self.h, P(mu_true), P(I0), C.c_uint64(seed), int(noisy), P(d)))
        return d

    # --- AM
    def am_init(self, d, I0, init_mu=None):
        self._d = np.ascontiguousarray(d, np.float64)
        self._I0 = np.ascontiguousarray(I0, np.float64)
        im = None if init_mu is None else np.ascontiguousarray(init_mu, np.float64)
        _chk(lib().orc_am_init(self.h, P(self._d), P(self._I0), P(im)))

    def am_iterate(self, n=1):
        recs = (Record * n)()
        _chk(lib().orc_am_iterate(self.h, int(n), recs))
        return [(r.iter, r.objective, r.elapsed_s, r.active_set, r.cum_updates) for r in recs]

    def am_get(self):
        mu = np.empty(self.N * self.nz)
        q = np.empty(self.M * self.nz)
        b = np.empty(self.N * self.nz)
        z0 = C.c_double()
        _chk(lib().orc_am_get(self.h, P(mu), P(q), C.byref(z0), P(b)))
        return dict(mu=mu, q=q, Z0=z0.value, b=b)

    # --- WAM
    def set_haar_dim(self, dim):
        _chk(lib().orc_set_haar_dim(self.h, int(dim)))

    def wam_init(self, d, I0, L, init_beta=None):
        self._d = np.ascontiguousarray(d, np.float64)
        self._I0 = np.ascontiguousarray(I0, np.float64)
        ib = None if init_beta is None else np.ascontiguousarray(init_beta, np.float64)
        _chk(lib().orc_wam_init(self.h, P(self._d), P(self._I0), int(L), P(ib)))
        self.L = L

    def wam_iterate(self, n=1):
        recs = (Record * n)()
        _chk(lib().orc_wam_iterate(self.h, int(n), recs))
        return [(r.iter, r.objective, r.elapsed_s, r.active_set, r.cum_updates) for r in recs]

    def wam_expand(self, factor=0.1):
        n = C.c_int64()
        _chk(lib().orc_wam_expand(self.h, C.c_double(factor), C.byref(n)))
        return n.value

    def wam_run(self, iters, schedule, factor=0.1):
        recs = (Record * iters)()
        s = np.ascontiguousarray(schedule, np.int32) if len(schedule) else np.zeros(1, np.int32)
        _chk(lib().orc_wam_run(self.h, int(iters), P(s, C.c_int), len(schedule), C.c_double(factor), recs))
        return [(r.iter, r.objective, r.elapsed_s, r.active_set, r.cum_updates) for r in recs]

    def wam_get(self):
        beta = np.empty(self.N * self.nz)
        mu = np.empty(self.N * self.nz)
        q = np.empty(self.M * self.nz)
        z0 = C.c_double()
        _chk(lib().orc_wam_get(self.h, P(beta), P(mu), P(q), C.byref(z0)))
        return dict(beta=beta, mu=mu, q=q, Z0=z0.value)

    def wam_tree(self):
        n = C.c_uint64()
        _chk(lib().orc_wam_tree(self.h, None, C.byref(n)))
        bits = np.empty(max(n.value, 1), np.uint8)
        _chk(lib().orc_wam_tree(self.h, P(bits, C.c_uint8), C.byref(n)))
        return bits[: n.value]

    def wam_stats(self):
        b = np.empty(self.N * self.nz)
        bp = np.empty(self.N * self.nz)
        bm = np.empty(self.N * self.nz)
        _chk(lib().orc_wam_stats(self.h, P(b), P(bp), P(bm)))
        return b, bp, bm

    def wam_counters(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        _chk(lib().orc_wam_counters(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return dict(cum_updates=a.value, degenerate=b.value, active_set=c.value)

    def wam_z0_rows(self):
        z = np.empty(self.M)
        _chk(lib().orc_wam_z0_rows(self.h, P(z)))
        return z

    def phi_column(self, L, z):
        n = C.c_uint64()
        _chk(lib().orc_phi_column(self.h, int(L), C.c_uint32(z), None, None, C.c_uint64(0), C.byref(n)))
        rows = np.empty(max(n.value, 1), np.uint32)
        vals = np.empty(max(n.value, 1))
        _chk(lib().orc_phi_column(self.h, int(L), C.c_uint32(z), P(rows, C.c_uint32), P(vals),
                                  C.c_uint64(n.value), C.byref(n)))
        return rows[: n.value], vals[: n.value]


def dwt2(x, nx, ny, L):
    x = np.ascontiguousarray(x, np.float64)
    ns = x.size // (nx * ny)
    out = np.empty_like(x)
    _chk(lib().orc_dwt2(nx, ny, ns, int(L), P(x), P(out)))
    return out


def idwt2(x, nx, ny, L):
    x = np.ascontiguousarray(x, np.float64)
    ns = x.size // (nx * ny)
    out = np.empty_like(x)
    _chk(lib().orc_idwt2(nx, ny, ns, int(L), P(x), P(out)))
    return out


def dwt3(x, nx, ny, nz, L):
    x = np.ascontiguousarray(x, np.float64)
    out = np.empty_like(x)
    _chk(lib().orc_dwt3(nx, ny, nz, int(L), P(x), P(out)))
    return out


def idwt3(x, nx, ny, nz, L):
    x = np.ascontiguousarray(x, np.float64)
    out = np.empty_like(x)
    _chk(lib().orc_idwt3(nx, ny, nz, int(L), P(x), P(out)))
    return out


def solve_update(b, bp, bm, Z0, beta):
    out = C.c_double()
    r = lib().orc_solve_update(b, bp, bm, Z0, beta, C.byref(out))
    if r < 0:
        raise OracleError(-r, lib().orc_last_error().decode())
    return r, out.value


def predicted_means(I0, l):
    I0 = np.ascontiguousarray(I0, np.float64)
    l = np.ascontiguousarray(l, np.float64)
    q = np.empty_like(l)
    _chk(lib().orc_predicted_means(C.c_uint64(l.size), P(I0), P(l), P(q)))
    return q


def i_divergence(d, q):
    d = np.ascontiguousarray(d, np.float64)
    q = np.ascontiguousarray(q, np.float64)
    out = C.c_double()
    _chk(lib().orc_i_divergence(C.c_uint64(d.size), P(d), P(q), C.byref(out)))
    return out.value


def rasterize(geom, prims, background=0.0):
    arr = (Primitive * max(len(prims), 1))()
    for i, p in enumerate(prims):
        arr[i] = Primitive(int(p["kind"]), *[float(p[k]) for k in
                                             ("cx", "cy", "cz", "ax", "ay", "az", "angle", "value")])
    mu = np.empty(geom.nx * geom.ny * geom.nz)
    _chk(lib().orc_rasterize(C.byref(geom), arr, len(prims), C.c_double(background), P(mu)))
    return mu


def uniform(seed, stream, k):
    return lib().orc_uniform(seed, stream, k)


def poisson(seed, stream, mean):
    return lib().orc_poisson(seed, stream, mean)


# ---------------------------------------------------------------- reference shim
class RefMatrix:
    """wamrec::SystemMatrix built by the unmodified reference headers."""

    def __init__(self, handle):
        self.h = handle
        R = reflib()
        rows, cols, nnz = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _chk(R.ref_dims(handle, C.byref(rows), C.byref(cols), C.byref(nnz)), R)
        self.M, self.N, self.nnz = rows.value, cols.value, nnz.value

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_free(self.h)

    @classmethod
    def build(cls, beam, nx, ny, nz, voxel, views, detectors, spacing, sod=0.0, sdd=0.0):
        R = reflib()
        h = C.c_void_p()
        _chk(R.ref_build(beam, nx, ny, nz, C.c_double(voxel), views, detectors, C.c_double(spacing),
                         C.c_double(sod), C.c_double(sdd), C.byref(h)), R)
        return cls(h)

    @classmethod
    def from_rays(cls, nx, ny, voxel, rays):
        R = reflib()
        rays = np.ascontiguousarray(rays, np.float64)
        h = C.c_void_p()
        _chk(R.ref_build_from_rays(nx, ny, C.c_double(voxel), C.c_uint64(rays.shape[0]), P(rays), C.byref(h)), R)
        return cls(h)

    def save(self, path):
        """wamrec::save_system_matrix (system_matrix.hpp:117-134)."""
        _chk(reflib().ref_save(self.h, os.fsencode(path)), reflib())

    @classmethod
    def load(cls, path):
        """wamrec::load_system_matrix (system_matrix.hpp:136-158)."""
        R = reflib()
        h = C.c_void_p()
        _chk(R.ref_load(os.fsencode(path), C.byref(h)), R)
        return cls(h)

    def csr(self):
        rp = np.empty(self.M + 1, np.uint64)
        ci = np.empty(self.nnz, np.uint32)
        v = np.empty(self.nnz, np.float64)
        _chk(reflib().ref_csr(self.h, P(rp, C.c_uint64), P(ci, C.c_uint32), P(v)), reflib())
        return rp, ci, v

    def csc(self):
        cp = np.empty(self.N + 1, np.uint64)
        ri = np.empty(self.nnz, np.uint32)
        v = np.empty(self.nnz, np.float64)
        _chk(reflib().ref_csc(self.h, P(cp, C.c_uint64), P(ri, C.c_uint32), P(v)), reflib())
        return cp, ri, v


def ref_trace(nx, ny, voxel, ray6, cap=4096):
    R = reflib()
    ray = np.ascontiguousarray(ray6, np.float64)
    ix = np.empty(cap, np.int32)
    iy = np.empty(cap, np.int32)
    ln = np.empty(cap)
    cnt = C.c_int()
    _chk(R.ref_trace(nx, ny, C.c_double(voxel), P(ray), cap, P(ix, C.c_int), P(iy, C.c_int), P(ln), C.byref(cnt)), R)
    n = cnt.value
    return ix[:n], iy[:n], ln[:n]


def ref_make_ray(beam, nx, ny, voxel, views, detectors, spacing, sod, sdd, view, det):
    R = reflib()
    out = np.empty(6)
    _chk(R.ref_make_ray(beam, nx, ny, C.c_double(voxel), views, detectors, C.c_double(spacing), C.c_double(sod),
                        C.c_double(sdd), view, det, P(out)), R)
    return out
