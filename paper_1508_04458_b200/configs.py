"""BASELINE.json configurations and their seeded synthetic phantoms.

The paper's SureScan x1000 / NIST Test Article A scan is proprietary and not
available: seeded synthetic phantoms with the
shapes, sizes and value ranges BASELINE.json prescribes stand in for it.
Pins: equiangular detector with delta-gamma =
2 asin(W/(2 SCD))/D (P1), SCD 500 mm / SDD 1000 mm for every config, axial
slices for 3D (P2), schedule floor(J k/(L+1)) (P4), global Z0 (P5),
per-channel gain for cfg4 (P6), fp32 storage (P7).

The phantom primitive lists are pure functions of the seed (splitmix64 counter
generator), so the GPU arm and the CPU baseline see identical inputs.
"""
from __future__ import annotations

import math

MASK = (1 << 64) - 1


def _mix(z):
    z = (z + 0x9E3779B97F4A7C15) & MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


class Rng:
    """Counter-based uniform stream (same mixer as the Poisson sampler)."""

    def __init__(self, seed, stream):
        self.seed, self.stream, self.k = seed, stream, 0

    def u(self, lo=0.0, hi=1.0):
        x = _mix(_mix(self.seed) ^ _mix((self.stream * 0x100000001B3 + self.k) & MASK))
        self.k += 1
        return lo + (hi - lo) * (((x >> 11) + 0.5) * 2.0 ** -53)

    def i(self, lo, hi):  # inclusive
        return lo + min(int(self.u() * (hi - lo + 1)), hi - lo)


def _prim(kind, cx, cy, ax, ay, angle, value, cz=0.0, az=1e9):
    return dict(kind=kind, cx=cx, cy=cy, cz=cz, ax=ax, ay=ay, az=az, angle=angle, value=value)


def bag_phantom(seed, W, nz_mm=None):
    """cfg1 family: ellipse 'bag' mu=0.02/mm with 6-10 random ellipses mu~U[0.005,0.05]
    and 2 small inclusions mu=0.5/mm (BASELINE.json configs[0])."""
    r = Rng(seed, 0xB46)
    s = W / 128.0
    prims = [_prim(0, 0.0, 0.0, 52.0 * s, 44.0 * s, r.u(0, math.pi), 0.02)]
    for _ in range(r.i(6, 10)):
        rad, th = r.u(0, 0.55), r.u(0, 2 * math.pi)
        prims.append(_prim(0, rad * 44.0 * s * math.cos(th), rad * 36.0 * s * math.sin(th), r.u(3, 12) * s,
                           r.u(3, 12) * s, r.u(0, math.pi), r.u(0.005, 0.05)))
    for _ in range(2):
        rad, th = r.u(0, 0.6), r.u(0, 2 * math.pi)
        rr = r.u(1.5, 3.0) * s
        prims.append(_prim(0, rad * 40.0 * s * math.cos(th), rad * 32.0 * s * math.sin(th), rr, rr, 0.0, 0.5))
    return prims


def luggage_phantom(seed, W, depth=None):
    """cfg2-cfg5 family: 'luggage' with 30-60 random ellipses and rectangles,
    mu~U[0,0.06]/mm, plus 4-8 metal-like inclusions mu~U[0.5,1.5]/mm.  With
    depth (mm) the primitives become ellipsoids / boxes spread over z."""
    r = Rng(seed, 0x1066)
    s = W / 256.0
    three_d = depth is not None
    zc = lambda: r.u(-0.4, 0.4) * depth if three_d else 0.0  # noqa: E731
    za = lambda lo, hi: r.u(lo, hi) * (depth / 64.0) if three_d else 1e9  # noqa: E731
    prims = [_prim(1, 0.0, 0.0, 105.0 * s, 80.0 * s, r.u(-0.2, 0.2), 0.012,
                   0.0, (0.45 * depth) if three_d else 1e9)]
    for _ in range(r.i(30, 60)):
        kind = r.i(0, 1)
        prims.append(_prim(kind, r.u(-85, 85) * s, r.u(-62, 62) * s, r.u(4, 28) * s, r.u(3, 20) * s,
                           r.u(0, math.pi), r.u(0.0, 0.06), zc(), za(4, 20)))
    for _ in range(r.i(4, 8)):
        kind = r.i(0, 1)
        prims.append(_prim(kind, r.u(-80, 80) * s, r.u(-58, 58) * s, r.u(1.0, 5.0) * s, r.u(1.0, 3.5) * s,
                           r.u(0, math.pi), r.u(0.5, 1.5), zc(), za(2, 6)))
    return prims


def schedule(J, L):
    """Pin P4: expansions at floor(J k / (L+1)), k = 1..L."""
    return [int(J * k // (L + 1)) for k in range(1, L + 1)]


CONFIGS = {
    # name: grid, voxel (mm), views, detectors, I0, L, J, seed, phantom
    "cfg1": dict(nx=128, ny=128, nz=1, voxel=1.0, views=180, detectors=256, I0=1e5, L=3, J=20, seed=1,
                 phantom="bag"),
    "cfg2": dict(nx=512, ny=512, nz=1, voxel=0.5, views=720, detectors=1024, I0=2e5, L=4, J=50, seed=2,
                 phantom="luggage"),
    "cfg3": dict(nx=512, ny=512, nz=64, voxel=1.0, views=720, detectors=1024, I0=2e5, L=3, J=30, seed=3,
                 phantom="luggage", haar=3),
    "cfg4": dict(nx=1024, ny=1024, nz=128, voxel=0.5, views=1440, detectors=1024, I0=1e5, L=4, J=40, seed=4,
                 phantom="luggage", gain=0.2, haar=3),
    "cfg5": dict(nx=512, ny=512, nz=64, voxel=1.0, views=720, detectors=1024, I0=2e5, L=0, J=30, seed=3,
                 phantom="luggage", algo="am"),
    # small parity cases (oracle finishes in seconds)
    "tiny": dict(nx=32, ny=32, nz=1, voxel=4.0, views=60, detectors=64, I0=1e5, L=3, J=12, seed=11,
                 phantom="bag"),
    "small": dict(nx=64, ny=64, nz=1, voxel=2.0, views=90, detectors=128, I0=1e5, L=3, J=16, seed=12,
                  phantom="bag"),
    "tiny3d": dict(nx=32, ny=32, nz=8, voxel=4.0, views=60, detectors=64, I0=1e5, L=3, J=12, seed=21,
                   phantom="luggage"),
    "small3d": dict(nx=64, ny=64, nz=40, voxel=4.0, views=72, detectors=96, I0=2e5, L=3, J=10, seed=22,
                    phantom="luggage"),
    # slab strides 16 and 32 (with 8 pad slices): the sharded small-slab layouts
    "tiny3d16": dict(nx=32, ny=32, nz=16, voxel=4.0, views=60, detectors=64, I0=1e5, L=3, J=10, seed=23,
                     phantom="luggage"),
    "tiny3d24": dict(nx=32, ny=32, nz=24, voxel=4.0, views=60, detectors=64, I0=1e5, L=3, J=10, seed=24,
                     phantom="luggage"),
    # 64 slices: 32 level-1 z-blocks, so the 3D Z walk splits level 1 across two warps
    "tiny3d64": dict(nx=32, ny=32, nz=64, voxel=4.0, views=60, detectors=64, I0=1e5, L=3, J=10, seed=25,
                     phantom="luggage"),
    "small_lug": dict(nx=128, ny=128, nz=1, voxel=2.0, views=120, detectors=192, I0=2e5, L=4, J=20, seed=13,
                      phantom="luggage"),
}


def get(name):
    c = dict(CONFIGS[name])
    c["name"] = name
    c.setdefault("algo", "wam")
    c.setdefault("haar", 2)   # 3: separable 3D Haar (pin P3, BASELINE cfg3/cfg4)
    c["schedule"] = schedule(c["J"], c["L"]) if c["L"] > 0 else []
    return c


def geometry(cfg, geometry_cls=None):
    """Geometry (pin P1 arc detector, SCD 500, SDD 1000) as kwargs or a ctypes struct."""
    W = cfg["nx"] * cfg["voxel"]
    dg = 2.0 * math.asin(W / (2.0 * 500.0)) / cfg["detectors"]
    kw = dict(nx=cfg["nx"], ny=cfg["ny"], nz=cfg["nz"], voxel=cfg["voxel"], views=cfg["views"],
              detectors=cfg["detectors"], beam=2, sod=500.0, sdd=1000.0, dgamma=dg)
    if geometry_cls is None:
        return kw
    return geometry_cls(kw["nx"], kw["ny"], kw["nz"], kw["voxel"], kw["detectors"], 0.0, kw["views"], None, 2,
                        500.0, 1000.0, dg)


def phantom(cfg):
    W = cfg["nx"] * cfg["voxel"]
    if cfg["phantom"] == "bag":
        return bag_phantom(cfg["seed"], W)
    depth = cfg["nz"] * cfg["voxel"] if cfg["nz"] > 1 else None
    return luggage_phantom(cfg["seed"], W, depth)


def incident(cfg, M_slice):
    """I0 per ray (z*M + y).  cfg4: seeded +-20 % per-channel gain (P6)."""
    import numpy as np
    nz, D = cfg["nz"], cfg["detectors"]
    I0 = np.full(M_slice * nz, float(cfg["I0"]))
    if cfg.get("gain"):
        r = Rng(cfg["seed"], 0x6A1)
        g = np.array([1.0 + r.u(-cfg["gain"], cfg["gain"]) for _ in range(D)])
        I0 *= np.tile(g, (M_slice // D) * nz)
    return I0
