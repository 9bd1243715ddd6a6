"""paper_1508_04458_b200 — B200-native alternating-minimization (AM) iteration of
arXiv 1508.04458 (multiresolution wavelet-domain AM for transmission CT).

The compute path is libwamgpu.so (CUDA kernels for sm_100a behind the C-ABI of
include/wamgpu.h).  This module is the Python mirror of the reference's
operator interface (proj/include/wamrec/),
used by the parity tests and the benchmark.  There is no CPU fallback: if the
extension is missing or no Blackwell GPU is present, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np

from . import configs  # noqa: F401  (re-export)

HERE = os.path.dirname(os.path.abspath(__file__))
LIBPATH = os.environ.get("WAMGPU_LIB") or os.path.join(HERE, "libwamgpu.so")   # WAMGPU_LIB: A/B against another build

BEAM_PARALLEL, BEAM_FAN_FLAT, BEAM_FAN_ARC = 0, 1, 2


# ---------------------------------------------------------------- errors
class Error(RuntimeError):
    """wamrec::Error (errors.hpp:9-13)."""


class ConfigError(Error):
    """wamrec::ConfigError (errors.hpp:17-20)."""


class ContractError(Error):
    """wamrec::ContractError (errors.hpp:22-25)."""


class NumericError(Error):
    """wamrec::NumericError (errors.hpp:27-30)."""


class IoError(Error):
    """wamrec::IoError (errors.hpp:32-35)."""


class CudaError(Error):
    """CUDA / NCCL failure (no reference equivalent)."""


_ERRS = {1: ConfigError, 2: ContractError, 3: NumericError, 4: IoError, 5: CudaError}

# symbols include/wamgpu.h declares (checked by tests/test_abi.py)
EXPORTED = [
    "wamgpu_version", "wamgpu_last_error", "wamgpu_create", "wamgpu_destroy", "wamgpu_nccl_unique_id",
    "wamgpu_set_comm", "wamgpu_set_geometry", "wamgpu_set_matrix_csr", "wamgpu_set_grid", "wamgpu_matrix_info",
    "wamgpu_get_matrix_csr", "wamgpu_get_matrix_csc", "wamgpu_forward_project", "wamgpu_back_project",
    "wamgpu_set_data", "wamgpu_am_init", "wamgpu_am_iterate", "wamgpu_wam_init", "wamgpu_wam_iterate",
    "wamgpu_wam_expand", "wamgpu_wam_run", "wamgpu_get_image", "wamgpu_get_beta", "wamgpu_get_q",
    "wamgpu_get_tree", "wamgpu_get_stats", "wamgpu_get_scalars", "wamgpu_get_z_rows", "wamgpu_get_timing",
    "wamgpu_set_kernel_timing", "wamgpu_rasterize", "wamgpu_simulate", "wamgpu_host_rays", "wamgpu_set_haar_dim",
    "wamgpu_p2p_export", "wamgpu_p2p_import", "wamgpu_selftest_fused_allreduce", "wamgpu_selftest_fused_back",
    "wamgpu_set_comm_local", "wamgpu_set_partition", "wamgpu_get_partition", "wamgpu_wam_expand_with", "wamgpu_simulate_device",
    "wamgpu_load_matrix_wamh", "wamgpu_save_matrix_wamh", "wamgpu_plan_partition",
    "wamgpu_set_projector", "wamgpu_get_projector", "wamgpu_debug_guards",
    "wamgpu_predicted_means", "wamgpu_i_divergence",
]
P2P_BLOB = 256   # WAMGPU_P2P_BLOB


# ---------------------------------------------------------------- C structs
_dp = C.POINTER(C.c_double)


class Geometry(C.Structure):
    """wamrec::ScanGeometry (geometry.hpp:21-68) as the C-ABI struct."""
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int), ("voxel_size", C.c_double),
                ("detectors", C.c_int), ("detector_spacing", C.c_double), ("views", C.c_int),
                ("view_angles", _dp), ("beam", C.c_int), ("source_to_center", C.c_double),
                ("source_to_detector", C.c_double), ("fan_angle_step", C.c_double)]

    def describe(self):
        return dict(nx=self.nx, ny=self.ny, nz=self.nz, voxel_size=self.voxel_size, detectors=self.detectors,
                    detector_spacing=self.detector_spacing, views=self.views, beam=self.beam,
                    source_to_center=self.source_to_center, source_to_detector=self.source_to_detector,
                    fan_angle_step=self.fan_angle_step)


class Plan(C.Structure):
    """wamgpu_plan: one rank's share of the rank grid (host-only arithmetic)."""
    _fields_ = [("view_groups", C.c_int), ("z_groups", C.c_int), ("view_group", C.c_int), ("z_group", C.c_int),
                ("row_begin", C.c_uint64), ("row_end", C.c_uint64), ("slab_begin", C.c_int),
                ("slab_slices", C.c_int), ("slab_stride", C.c_int), ("split_update", C.c_int),
                ("own_row_begin", C.c_int), ("own_rows", C.c_int)]

    def asdict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


def debug_guards():
    """(checked, bad, message): guard bands of every live device allocation
    (WAMGPU_GUARD=1 must be in the environment before the library allocates)."""
    n, b = C.c_uint64(), C.c_uint64()
    _chk(load().wamgpu_debug_guards(C.byref(n), C.byref(b)), None)
    return n.value, b.value, (load().wamgpu_last_error(None).decode() if b.value else "")


def plan_partition(g, rank, nranks, view_groups=0, algo="wam", haar_dim=3, levels=0):
    """The rank grid of wamgpu_set_partition / set_geometry for `rank` of
    `nranks`, computed on the host (no GPU needed)."""
    out = Plan()
    _chk(load().wamgpu_plan_partition(C.byref(g), int(rank), int(nranks), int(view_groups),
                                      1 if algo == "am" else 2, int(haar_dim), int(levels), C.byref(out)))
    return out.asdict()


class Primitive(C.Structure):
    _fields_ = [("kind", C.c_int)] + [(n, C.c_double) for n in
                                      ("cx", "cy", "cz", "ax", "ay", "az", "angle", "value")]


class Record(C.Structure):
    """ConvergenceRecord."""
    _fields_ = [("iter", C.c_int), ("objective", C.c_double), ("elapsed_s", C.c_double),
                ("active_set", C.c_int64), ("cum_updates", C.c_int64)]


class Timing(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("total_ms", "fwd_ms", "back_ms", "split_ms", "update_ms",
                                          "expand_ms", "comm_ms")] + \
               [(n, C.c_int64) for n in ("fwd_launches", "back_launches", "split_launches", "update_launches",
                                         "expand_events", "kernel_launches", "split_nnz")] + \
               [("phi_ms", C.c_double), ("phi_launches", C.c_int64), ("coarse_fwd_ms", C.c_double),
                ("coarse_back_ms", C.c_double), ("coarse_fwd_launches", C.c_int64),
                ("coarse_back_launches", C.c_int64), ("proj_updates", C.c_int64), ("split_entries", C.c_int64)]

    def asdict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


def make_parallel_geometry(nx, ny, nz, voxel_size, views, detectors, detector_spacing):
    """geometry.hpp:77-92 (views over [0, pi))."""
    return Geometry(nx, ny, nz, voxel_size, detectors, detector_spacing, views, None, BEAM_PARALLEL, 0.0, 0.0, 0.0)


def make_fan_geometry(nx, ny, nz, voxel_size, views, detectors, detector_spacing, source_to_center,
                      source_to_detector):
    """geometry.hpp:95-112 (flat detector, views over [0, 2pi))."""
    return Geometry(nx, ny, nz, voxel_size, detectors, detector_spacing, views, None, BEAM_FAN_FLAT,
                    source_to_center, source_to_detector, 0.0)


def make_arc_geometry(nx, ny, nz, voxel_size, views, detectors, source_to_center=500.0,
                      source_to_detector=1000.0, fan_angle_step=None):
    """Equiangular ("curved") detector, pin P1: delta-gamma = 2 asin(W / (2 SCD)) / D."""
    if fan_angle_step is None:
        W = nx * voxel_size
        fan_angle_step = 2.0 * math.asin(W / (2.0 * source_to_center)) / detectors
    return Geometry(nx, ny, nz, voxel_size, detectors, 0.0, views, None, BEAM_FAN_ARC, source_to_center,
                    source_to_detector, fan_angle_step)


# ---------------------------------------------------------------- library
_lib = None


def load():
    """Load libwamgpu.so; raises loudly when the extension has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIBPATH):
            raise ImportError(f"{LIBPATH} missing: run `python -m paper_1508_04458_b200.build` "
                              "(there is no CPU fallback)")
        lib = C.CDLL(LIBPATH)
        lib.wamgpu_last_error.restype = C.c_char_p
        lib.wamgpu_last_error.argtypes = [C.c_void_p]
        lib.wamgpu_destroy.argtypes = [C.c_void_p]
        _lib = lib
    return _lib


def _chk(rc, ctx=None):
    if rc != 0:
        msg = load().wamgpu_last_error(ctx).decode()
        raise _ERRS.get(rc, Error)(msg)


def _p(a, ct=C.c_double):
    return None if a is None else a.ctypes.data_as(C.POINTER(ct))


def _records(arr):
    return [dict(iter=r.iter, objective=r.objective, elapsed_s=r.elapsed_s, active_set=r.active_set,
                 cum_updates=r.cum_updates) for r in arr]


def selftest_fused_allreduce(partials, epochs=2, device=0):
    """R logical ranks of the fused all-reduce in one cooperative grid on one
    GPU: partials (R, n) -> every rank's result (R, n)."""
    p = np.ascontiguousarray(partials, np.float64)
    R, n = p.shape
    out = np.empty_like(p)
    _chk(load().wamgpu_selftest_fused_allreduce(int(device), int(R), C.c_uint64(n), _p(p), _p(out), int(epochs)))
    return out


def selftest_fused_back(ctxs, ws, extras=None):
    """The fused back projection + all-reduce over R contexts (context k plays
    rank k with its own row shard) on one GPU: returns (R, 2N)."""
    R = len(ctxs)
    hs = (C.c_void_p * R)(*[c.h for c in ctxs])
    wk = [np.ascontiguousarray(w, np.float64) for w in ws]
    wp = (C.POINTER(C.c_double) * R)(*[_p(w) for w in wk])
    ek = None
    ep = None
    if extras is not None:
        ek = [np.ascontiguousarray(e, np.float64) for e in extras]
        ep = (C.POINTER(C.c_double) * R)(*[_p(e) for e in ek])
    out = np.empty((R, 2 * ctxs[0].N), np.float64)
    _chk(load().wamgpu_selftest_fused_back(hs, int(R), wp, ep, _p(out)))
    return out


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _chk(load().wamgpu_nccl_unique_id(buf))
    return buf.raw


class Context:
    """One GPU.  Mirrors the reference's reconstruct/iterate API (SPEC.md:63-98,
    300-308, 353-389) over the C-ABI; host numpy arrays in and out."""

    def __init__(self, device=0):
        lib = load()
        h = C.c_void_p()
        _chk(lib.wamgpu_create(int(device), C.byref(h)))
        self.h = h
        self.M = self.N = self.nnz = self.row0 = self.row1 = None
        self.nz = 1

    def close(self):
        if getattr(self, "h", None):
            load().wamgpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- setup
    def set_comm(self, uid: bytes, rank: int, nranks: int):
        _chk(load().wamgpu_set_comm(self.h, C.c_char_p(uid) if uid else None, int(rank), int(nranks)), self.h)

    def set_comm_local(self, group: int, rank: int, nranks: int):
        """In-process ranks (one host thread per context) joined under `group`;
        group < 0: a detached shard (this rank's share alone, no exchange)."""
        _chk(load().wamgpu_set_comm_local(self.h, int(group), int(rank), int(nranks)), self.h)

    def set_partition(self, view_groups: int):
        """Rank grid: view_groups x (nranks / view_groups) z groups (3D); 0 = default."""
        _chk(load().wamgpu_set_partition(self.h, int(view_groups)), self.h)

    def set_projector(self, kind: int):
        """3D forward projector: 0 = slab SpMM over the stored in-plane matrix,
        1 = on the fly (rays re-traced every pass, image tiles staged by TMA)."""
        _chk(load().wamgpu_set_projector(self.h, int(kind)), self.h)

    def projector(self) -> int:
        """0 stored matrix, 1 on the fly requested, 2 on the fly active, -1 rejected."""
        v = C.c_int()
        _chk(load().wamgpu_get_projector(self.h, C.byref(v)), self.h)
        return v.value

    def partition(self):
        v = [C.c_int() for _ in range(4)]
        _chk(load().wamgpu_get_partition(self.h, *[C.byref(x) for x in v]), self.h)
        return dict(view_groups=v[0].value, z_groups=v[1].value, slab_begin=v[2].value, slab_slices=v[3].value)

    def p2p_export(self) -> bytes:
        """This rank's CUDA IPC handles for the fused back projection +
        all-reduce over NVLink peer memory (after set_comm and the matrix)."""
        buf = C.create_string_buffer(P2P_BLOB)
        _chk(load().wamgpu_p2p_export(self.h, buf), self.h)
        return buf.raw

    def p2p_import(self, blobs: bytes) -> bool:
        """blobs: every rank's p2p_export() concatenated in rank order.  Runs a
        collective self-check; True when the fused path is active."""
        ok = C.c_int(0)
        _chk(load().wamgpu_p2p_import(self.h, C.c_char_p(blobs), C.byref(ok)), self.h)
        return bool(ok.value)

    def _info(self):
        M, N, nnz, r0, r1 = (C.c_uint64() for _ in range(5))
        _chk(load().wamgpu_matrix_info(self.h, C.byref(M), C.byref(N), C.byref(nnz), C.byref(r0), C.byref(r1)),
             self.h)
        self.M, self.N, self.nnz, self.row0, self.row1 = M.value, N.value, nnz.value, r0.value, r1.value

    def set_geometry(self, g: Geometry):
        """build_system_matrix (projector.hpp:126-148) on the device."""
        _chk(load().wamgpu_set_geometry(self.h, C.byref(g)), self.h)
        self.geom = g
        self.nz = g.nz
        self._info()

    def set_grid(self, nx, ny, nz=1):
        _chk(load().wamgpu_set_grid(self.h, int(nx), int(ny), int(nz)), self.h)
        self.nz = nz

    def set_matrix_csr(self, row_ptr, col_idx, values, cols):
        """SystemMatrix(rows, cols, row_ptr, col_idx, values) (system_matrix.hpp:24-35)."""
        rp = np.ascontiguousarray(row_ptr, np.uint64)
        ci = np.ascontiguousarray(col_idx, np.uint32)
        v = np.ascontiguousarray(values, np.float64)
        _chk(load().wamgpu_set_matrix_csr(self.h, C.c_uint64(rp.size - 1), C.c_uint64(cols), C.c_uint64(v.size),
                                          _p(rp, C.c_uint64), _p(ci, C.c_uint32), _p(v)), self.h)
        self._info()

    def load_matrix_wamh(self, path):
        """load_system_matrix (system_matrix.hpp:136-158): WAMH v1 (reference) or v2."""
        _chk(load().wamgpu_load_matrix_wamh(self.h, os.fsencode(path)), self.h)
        self._info()

    def save_matrix_wamh(self, path, version=2, with_csc=False):
        """save_system_matrix (system_matrix.hpp:117-134): v1 = reference layout,
        v2 = fp32 device layout (optionally with the CSC mirror)."""
        _chk(load().wamgpu_save_matrix_wamh(self.h, os.fsencode(path), int(version), int(bool(with_csc))), self.h)

    def matrix_csr(self):
        rp = np.empty(self.row1 - self.row0 + 1, np.uint64)
        ci = np.empty(max(self.nnz, 1), np.uint32)
        v = np.empty(max(self.nnz, 1), np.float32)
        _chk(load().wamgpu_get_matrix_csr(self.h, _p(rp, C.c_uint64), _p(ci, C.c_uint32), _p(v, C.c_float)),
             self.h)
        return rp, ci[: self.nnz], v[: self.nnz]

    def matrix_csc(self):
        cp = np.empty(self.N + 1, np.uint64)
        ri = np.empty(max(self.nnz, 1), np.uint32)
        v = np.empty(max(self.nnz, 1), np.float32)
        _chk(load().wamgpu_get_matrix_csc(self.h, _p(cp, C.c_uint64), _p(ri, C.c_uint32), _p(v, C.c_float)),
             self.h)
        return cp, ri[: self.nnz], v[: self.nnz]

    # ---- core-model
    def forward_project(self, mu):
        mu = np.ascontiguousarray(mu, np.float64)
        out = np.empty((self.row1 - self.row0) * self.nz)
        _chk(load().wamgpu_forward_project(self.h, _p(mu), _p(out)), self.h)
        return out

    def back_project(self, w):
        w = np.ascontiguousarray(w, np.float64)
        out = np.empty(self.N * self.nz)
        _chk(load().wamgpu_back_project(self.h, _p(w), _p(out)), self.h)
        return out

    # ---- core-model, standalone on caller vectors
    def predicted_means(self, I0, l):
        I0 = np.ascontiguousarray(I0, np.float64).ravel()
        l = np.ascontiguousarray(l, np.float64).ravel()
        if I0.size != l.size:
            raise ContractError("predicted_means: length mismatch")
        q = np.empty(l.size)
        _chk(load().wamgpu_predicted_means(self.h, C.c_uint64(l.size), _p(I0), _p(l), _p(q)), self.h)
        return q

    def i_divergence(self, d, q):
        d = np.ascontiguousarray(d, np.float64).ravel()
        q = np.ascontiguousarray(q, np.float64).ravel()
        if d.size != q.size:
            raise ContractError("i_divergence: length mismatch")
        out = C.c_double(0.0)
        _chk(load().wamgpu_i_divergence(self.h, C.c_uint64(d.size), _p(d), _p(q), C.byref(out)), self.h)
        return out.value

    def set_data(self, d, I0):
        self._d = np.ascontiguousarray(d, np.float64)
        self._I0 = np.ascontiguousarray(I0, np.float64)
        _chk(load().wamgpu_set_data(self.h, _p(self._d), _p(self._I0)), self.h)

    # ---- AM baseline
    def am_init(self, init_mu=None):
        m = None if init_mu is None else np.ascontiguousarray(init_mu, np.float64)
        _chk(load().wamgpu_am_init(self.h, _p(m)), self.h)

    def am_iterate(self, n=1):
        recs = (Record * max(n, 1))()
        _chk(load().wamgpu_am_iterate(self.h, int(n), recs), self.h)
        return _records(recs[:n])

    # ---- wavelet AM
    def set_haar_dim(self, dim):
        """2: per-slice 2D Haar (SPEC model); 3: separable 3D Haar (pin P3)."""
        _chk(load().wamgpu_set_haar_dim(self.h, int(dim)), self.h)

    def wam_init(self, levels, init_beta=None):
        b = None if init_beta is None else np.ascontiguousarray(init_beta, np.float64)
        _chk(load().wamgpu_wam_init(self.h, int(levels), _p(b)), self.h)
        self.levels = levels

    def wam_iterate(self, n=1):
        recs = (Record * max(n, 1))()
        _chk(load().wamgpu_wam_iterate(self.h, int(n), recs), self.h)
        return _records(recs[:n])

    def wam_expand(self, factor=0.1, add_tree=None):
        """expand_tree; add_tree: blocks of another tree (get_tree
        layout) activated together with the criterion's marks."""
        n = C.c_int64()
        if add_tree is None:
            _chk(load().wamgpu_wam_expand(self.h, C.c_double(factor), C.byref(n)), self.h)
        else:
            t = np.ascontiguousarray(add_tree, np.uint8)
            _chk(load().wamgpu_wam_expand_with(self.h, C.c_double(factor), _p(t, C.c_uint8), C.c_uint64(t.size),
                                               C.byref(n)), self.h)
        return n.value

    def wam_run(self, iters, schedule=(), factor=0.1):
        recs = (Record * max(iters, 1))()
        s = np.ascontiguousarray(list(schedule) or [0], np.int32)
        _chk(load().wamgpu_wam_run(self.h, int(iters), _p(s, C.c_int), len(schedule), C.c_double(factor), recs),
             self.h)
        return _records(recs[:iters])

    # ---- state
    def image(self):
        out = np.empty(self.N * self.nz)
        _chk(load().wamgpu_get_image(self.h, _p(out)), self.h)
        return out

    def beta(self):
        out = np.empty(self.N * self.nz)
        _chk(load().wamgpu_get_beta(self.h, _p(out)), self.h)
        return out

    def q(self):
        out = np.empty((self.row1 - self.row0) * self.nz)
        _chk(load().wamgpu_get_q(self.h, _p(out)), self.h)
        return out

    def tree(self):
        n = C.c_uint64()
        _chk(load().wamgpu_get_tree(self.h, None, C.byref(n)), self.h)
        out = np.empty(max(n.value, 1), np.uint8)
        _chk(load().wamgpu_get_tree(self.h, _p(out, C.c_uint8), C.byref(n)), self.h)
        return out[: n.value]

    def stats(self):
        n = self.N * self.nz
        b, bp, bm = np.empty(n), np.empty(n), np.empty(n)
        _chk(load().wamgpu_get_stats(self.h, _p(b), _p(bp), _p(bm)), self.h)
        return b, bp, bm

    def scalars(self):
        z0 = C.c_double()
        cum, deg, act = C.c_int64(), C.c_int64(), C.c_int64()
        _chk(load().wamgpu_get_scalars(self.h, C.byref(z0), C.byref(cum), C.byref(deg), C.byref(act)), self.h)
        return dict(Z0=z0.value, cum_updates=cum.value, degenerate=deg.value, active_set=act.value)

    def z_rows(self):
        out = np.empty(self.row1 - self.row0)
        _chk(load().wamgpu_get_z_rows(self.h, _p(out)), self.h)
        return out

    def timing(self):
        t = Timing()
        _chk(load().wamgpu_get_timing(self.h, C.byref(t)), self.h)
        return t.asdict()

    def set_kernel_timing(self, on=True):
        _chk(load().wamgpu_set_kernel_timing(self.h, int(bool(on))), self.h)


# ---------------------------------------------------------------- phantom-sim
def rasterize(g: Geometry, prims, background=0.0):
    """rasterize_phantom."""
    arr = (Primitive * max(len(prims), 1))()
    for i, p in enumerate(prims):
        arr[i] = Primitive(int(p["kind"]), *[float(p[k]) for k in ("cx", "cy", "cz", "ax", "ay", "az", "angle",
                                                                     "value")])
    mu = np.empty(g.nx * g.ny * g.nz)
    _chk(load().wamgpu_rasterize(C.byref(g), arr, len(prims), C.c_double(background), _p(mu)))
    return mu


def simulate(g: Geometry, mu_true, I0, seed, noisy=True, threads=0):
    """simulate_counts: f64 host, seeded counter RNG."""
    mu_true = np.ascontiguousarray(mu_true, np.float64)
    I0 = np.ascontiguousarray(I0, np.float64)
    d = np.empty(I0.size)
    _chk(load().wamgpu_simulate(C.byref(g), _p(mu_true), _p(I0), C.c_uint64(seed), int(noisy), int(threads),
                                _p(d)))
    return d


def simulate_device(g: Geometry, mu_true, I0, seed, noisy=True, device=0):
    """simulate_counts on a CUDA device: the host simulator's trace, sums and
    counter-based Poisson generator, one warp per ray."""
    mu_true = np.ascontiguousarray(mu_true, np.float64)
    I0 = np.ascontiguousarray(I0, np.float64)
    d = np.empty(I0.size)
    _chk(load().wamgpu_simulate_device(int(device), C.byref(g), _p(mu_true), _p(I0), C.c_uint64(seed), int(noisy),
                                       _p(d)))
    return d


def host_rays(g: Geometry):
    r = np.empty((g.views * g.detectors, 6))
    _chk(load().wamgpu_host_rays(C.byref(g), _p(r)))
    return r
