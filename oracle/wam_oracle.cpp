// wam_oracle.cpp — CPU ORACLE for the wavelet-domain AM iteration of arXiv 1508.04458.
//
// TEST INFRASTRUCTURE ONLY.  Loaded exclusively by tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs, as the checker.  The
// product library (libwamgpu.so) never links, loads or calls anything here.
//
// What it restates (all citations relative to /root/reference/):
//   * geometry defaults/validation ............ proj/include/wamrec/geometry.hpp:51-112
//   * make_ray (parallel, flat fan) ........... proj/include/wamrec/projector.hpp:22-49
//     + equiangular arc detector ............. pin P1
//   * clip_axis / trace_ray (Siddon) .......... projector.hpp:52-119
//   * build_system_matrix (row = v*D + k) ..... projector.hpp:123-148
//   * CSC mirror by counting sort ............. system_matrix.hpp:61-75
//   * parallel_for ............................ parallel.hpp:11-41
//   * forward/back projection, Beer, I-div .... SPEC.md:63-98, 106-113
//   * phantom rasterisation, Poisson data ..... SPEC.md:144-161, 167-173
//   * orthonormal 2D Haar (Mallat layout) ..... SPEC.md:212-229, 265-266
//   * footprints / phi = H*Omega*e_z .......... SPEC.md:230-247
//   * active tree + expand_tree ............... SPEC.md:197-203, 248-256, 267-268
//   * AM baseline ............................. SPEC.md:292-318, 330
//   * root solver (errata E1, E2) ............. SPEC.md:362-370, 400, 403
//   * wam_iterate / run ....................... SPEC.md:338-389, 399-404
//
// Parity pinning: the system matrix (ray table + Siddon) is pinned bit-for-bit
// against the reference headers compiled verbatim (oracle/_ref, built by
// oracle/Makefile from /root/reference).  The iteration itself has no
// executable reference: it is pinned by the SPEC's scalar known-answer tests
// (with errata E1/E2 applied) and its property tests (adjoint, Parseval,
// monotone I-divergence, reduction equivalence, root-vs-bisection, Z0
// validity, expansion-oracle set equality); see tests/test_oracle_*.py.
//
// Two storage modes (pin P7):
//   mirror = 0  reference-faithful f64 storage everywhere.  b+/b- come from a
//               direct per-(ray, coefficient) signed split over exact phi.
//   mirror = 1  fp32 storage of h, mu, beta, q, d, I0 with fp64 accumulation,
//               computing b+/b- the way the GPU does (b+ = [Omega^T H^T q](z) - b-,
//               b- gathered from explicit negative phi columns), so the active
//               tree can be compared bit-for-bit with the GPU.
//
// Build: -std=c++20 -O3 -ffp-contract=off (FMA contraction changes 16% of h
// bitwise).
#include "wam_oracle.h"

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numbers>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace orc {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};
static Error config_error(const std::string& w) { return Error(ORC_ERR_CONFIG, w); }
static Error contract_error(const std::string& w) { return Error(ORC_ERR_CONTRACT, w); }
static Error numeric_error(const std::string& w) { return Error(ORC_ERR_NUMERIC, w); }

static thread_local std::string g_err;

// ---- parallel.hpp:11-41 restated: static contiguous chunks, disjoint writes only.
static int resolve_threads(int requested) {
    if (requested > 0) return requested;
    unsigned hw = std::thread::hardware_concurrency();
    return hw == 0 ? 1 : static_cast<int>(hw);
}
template <typename Fn>
static void parallel_for(std::size_t n, int threads, Fn&& fn) {
    threads = resolve_threads(threads);
    if (n == 0) return;
    if (threads <= 1 || n < 2) { fn(std::size_t{0}, n, 0); return; }
    std::size_t nb = std::min<std::size_t>(static_cast<std::size_t>(threads), n);
    std::size_t chunk = (n + nb - 1) / nb;
    std::vector<std::thread> pool;
    for (std::size_t b = 0; b < nb; ++b) {
        std::size_t lo = b * chunk, hi = std::min(n, lo + chunk);
        if (lo >= hi) break;
        pool.emplace_back([&fn, lo, hi, b] { fn(lo, hi, (int)b); });
    }
    for (auto& t : pool) t.join();
}

// ---- geometry.hpp:21-112 restated (plus pin P1 arc detector).
struct Geom {
    int nx = 0, ny = 0, nz = 1;
    double voxel = 1.0;
    int detectors = 0;
    double spacing = 1.0;
    std::vector<double> angles;
    int beam = 0;
    double sod = 0.0, sdd = 0.0, dgamma = 0.0;
    int views() const { return (int)angles.size(); }
    double width() const { return nx * voxel; }   // geometry.hpp:44
    double height() const { return ny * voxel; }  // geometry.hpp:45
};

static std::vector<double> uniform_angles(int views, double arc) {  // geometry.hpp:70-74
    std::vector<double> a((std::size_t)views);
    for (int v = 0; v < views; ++v) a[v] = arc * v / views;
    return a;
}

static Geom make_geom(const orc_geometry* c) {
    if (!c) throw contract_error("geometry: null");
    Geom g;
    g.nx = c->nx; g.ny = c->ny; g.nz = c->nz; g.voxel = c->voxel_size;
    g.detectors = c->detectors; g.spacing = c->detector_spacing; g.beam = c->beam;
    g.sod = c->source_to_center; g.sdd = c->source_to_detector; g.dgamma = c->fan_angle_step;
    if (c->views < 1) throw config_error("geometry: at least one view required");
    if (c->view_angles) g.angles.assign(c->view_angles, c->view_angles + c->views);
    else g.angles = uniform_angles(c->views, g.beam == 0 ? std::numbers::pi : 2.0 * std::numbers::pi);
    // validate(): geometry.hpp:51-67
    if (g.nx < 4 || g.ny < 4) throw config_error("geometry: nx and ny must be >= 4");
    if (g.nz < 1) throw config_error("geometry: nz must be >= 1");
    if (!(g.voxel > 0.0)) throw config_error("geometry: voxel_size must be positive");
    if (g.detectors < 1) throw config_error("geometry: at least one detector required");
    if (g.beam != 2 && !(g.spacing > 0.0)) throw config_error("geometry: detector_spacing must be positive");
    for (double a : g.angles)
        if (!std::isfinite(a)) throw config_error("geometry: non-finite view angle");
    if (g.beam < 0 || g.beam > 2) throw config_error("geometry: unknown beam type");
    if (g.beam != 0) {
        if (!(g.sod > 0.0)) throw config_error("geometry: source_to_center must be positive");
        if (!(g.sdd > g.sod)) throw config_error("geometry: source_to_detector must exceed source_to_center");
    }
    if (g.beam == 2 && !(g.dgamma > 0.0)) throw config_error("geometry: fan_angle_step must be positive");
    return g;
}

struct Ray { double ox, oy, dx, dy, tmin, tmax; };

// projector.hpp:22-49 (beam 0/1) with the identical operation order; beam 2 is
// the pinned equiangular array: same source, direction rotated by gamma_k from
// the central ray, t in [0, SDD].
static Ray make_ray(const Geom& g, int view, int det) {
    const double theta = g.angles[view];
    const double c = std::cos(theta), s = std::sin(theta);
    Ray r{};
    if (g.beam == 0) {
        const double u = (det - 0.5 * (g.detectors - 1)) * g.spacing;
        r.ox = -s * u; r.oy = c * u; r.dx = c; r.dy = s;
        r.tmin = -std::numeric_limits<double>::max();
        r.tmax = std::numeric_limits<double>::max();
    } else if (g.beam == 1) {
        const double u = (det - 0.5 * (g.detectors - 1)) * g.spacing;
        const double sx = g.sod * c, sy = g.sod * s;
        const double px = sx - g.sdd * c - s * u;
        const double py = sy - g.sdd * s + c * u;
        const double len = std::hypot(px - sx, py - sy);
        r.ox = sx; r.oy = sy; r.dx = (px - sx) / len; r.dy = (py - sy) / len;
        r.tmin = 0.0; r.tmax = len;
    } else {
        const double gam = (det - 0.5 * (g.detectors - 1)) * g.dgamma;
        const double cg = std::cos(gam), sg = std::sin(gam);
        r.ox = g.sod * c; r.oy = g.sod * s;
        r.dx = -c * cg - s * sg;
        r.dy = -s * cg + c * sg;
        r.tmin = 0.0; r.tmax = g.sdd;
    }
    return r;
}

// projector.hpp:52-60
static bool clip_axis(double o, double d, double lo, double hi, double& tmin, double& tmax) {
    if (d == 0.0) return o >= lo && o <= hi;
    double t0 = (lo - o) / d, t1 = (hi - o) / d;
    if (t0 > t1) std::swap(t0, t1);
    if (t0 > tmin) tmin = t0;
    if (t1 < tmax) tmax = t1;
    return tmin < tmax;
}

// projector.hpp:64-119, same operation order (exactness needs -ffp-contract=off).
template <typename Emit>
static void trace(const Geom& g, const Ray& ray, Emit&& emit) {
    const double h = g.voxel;
    const double xmin = -0.5 * g.width();
    const double ymin = -0.5 * g.height();
    double tmin = ray.tmin, tmax = ray.tmax;
    if (!clip_axis(ray.ox, ray.dx, xmin, xmin + g.width(), tmin, tmax)) return;
    if (!clip_axis(ray.oy, ray.dy, ymin, ymin + g.height(), tmin, tmax)) return;
    if (!(tmax > tmin)) return;
    auto cell = [](double pos, double origin, double edge, int n) {
        int i = static_cast<int>(std::floor((pos - origin) / edge));
        return std::clamp(i, 0, n - 1);
    };
    const double ex = ray.ox + tmin * ray.dx;
    const double ey = ray.oy + tmin * ray.dy;
    int ix = cell(ex, xmin, h, g.nx), iy = cell(ey, ymin, h, g.ny);
    const int step_x = ray.dx > 0.0 ? 1 : -1, step_y = ray.dy > 0.0 ? 1 : -1;
    const double big = std::numeric_limits<double>::max();
    const double dt_x = ray.dx != 0.0 ? h / std::abs(ray.dx) : big;
    const double dt_y = ray.dy != 0.0 ? h / std::abs(ray.dy) : big;
    double next_x = big, next_y = big;
    if (ray.dx != 0.0) { double e = xmin + (ray.dx > 0.0 ? ix + 1 : ix) * h; next_x = (e - ray.ox) / ray.dx; }
    if (ray.dy != 0.0) { double e = ymin + (ray.dy > 0.0 ? iy + 1 : iy) * h; next_y = (e - ray.oy) / ray.dy; }
    double t = tmin;
    while (t < tmax) {
        double t_stop = std::min({next_x, next_y, tmax});
        double len = t_stop - t;
        if (len > 0.0) emit(ix, iy, len);
        if (t_stop >= tmax) break;
        if (next_x <= t_stop) { ix += step_x; next_x += dt_x; if (ix < 0 || ix >= g.nx) break; }
        if (next_y <= t_stop) { iy += step_y; next_y += dt_y; if (iy < 0 || iy >= g.ny) break; }
        t = t_stop;
    }
}

// ---- splitmix64 counter RNG (counter-based, per-ray streams)
static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline double uniform(uint64_t seed, uint64_t stream, uint64_t k) {
    uint64_t x = mix64(mix64(seed) ^ mix64(stream * 0x100000001B3ull + k));
    return ((double)(x >> 11) + 0.5) * 0x1.0p-53;  // open interval (0,1)
}
// Poisson sampling: inversion for mean < 12, PTRS transformed rejection
// (Hoermann 1993) otherwise.
static double poisson(uint64_t seed, uint64_t stream, double m) {
    if (!(m >= 0.0) || !std::isfinite(m)) throw numeric_error("simulate: invalid Poisson mean");
    if (m == 0.0) return 0.0;
    if (m < 12.0) {
        double u = uniform(seed, stream, 0);
        double p = std::exp(-m), F = p;
        double k = 0.0;
        while (u > F && k < 1000.0) { k += 1.0; p *= m / k; F += p; }
        return k;
    }
    const double slam = std::sqrt(m), loglam = std::log(m);
    const double b = 0.931 + 2.53 * slam;
    const double a = -0.059 + 0.02483 * b;
    const double invalpha = 1.1239 + 1.1328 / (b - 3.4);
    const double vr = 0.9277 - 3.6224 / (b - 2.0);
    for (uint64_t j = 0;; ++j) {
        double U = uniform(seed, stream, 2 * j + 1) - 0.5;
        double V = uniform(seed, stream, 2 * j + 2);
        double us = 0.5 - std::fabs(U);
        double k = std::floor((2.0 * a / us + b) * U + m + 0.43);
        if (us >= 0.07 && V <= vr) return k;
        if (k < 0.0 || (us < 0.013 && V > us)) continue;
        if (std::log(V) + std::log(invalpha) - std::log(a / (us * us) + b) <=
            -m + k * loglam - std::lgamma(k + 1.0))
            return k;
    }
}

}  // namespace orc

using namespace orc;

// Psi lists of one level (3D model): per in-plane block b, the rays crossing b
// (ascending) with psi_A, psi_H, psi_V, psi_D (2^-l scaled quadrant
// combinations of phi_walk; fp32-rounded in mirror mode, exact f64 otherwise).
struct PsiLevel {
    std::vector<uint64_t> ptr;                 // [b + 1]
    std::vector<uint32_t> ray;                 // [entry]
    std::vector<std::array<double, 4>> val;    // [entry]
};

struct orc_problem {
    Geom g;
    bool mirror = false;
    // slim (ORC_SLIM): CSR only, no exact-h copy and no CSC mirror; h stored as
    // fp32 in mirror mode.  Back projection is then a ray-ordered CSR scatter
    // per slice group, which adds the terms of every voxel in the same
    // (ascending-ray) order as the CSC gather, so results are bit-identical.
    bool slim = false;
    int threads = 0;
    uint64_t Ms = 0, Ns = 0;
    int nz = 1;
    std::vector<Ray> rays;
    std::vector<uint64_t> rp;
    std::vector<uint32_t> ci;
    std::vector<double> hexact, hv;  // hv = stored h (fp32-rounded in mirror mode)
    std::vector<float> hv32;         // slim + mirror: stored h as fp32
    std::vector<uint64_t> cp;
    std::vector<uint32_t> ri;
    std::vector<double> cv;
    inline double hvk(uint64_t k) const { return hv32.empty() ? hv[k] : (double)hv32[k]; }
    std::vector<double> d, I0;  // stored data
    // AM state
    bool am_ready = false;
    std::vector<double> am_mu, am_q, am_b;
    double am_Z0 = 0.0;
    int am_iter = 0;
    bool am_clamp = true;
    // WAM state
    bool wam_ready = false;
    int L = 0;
    std::vector<std::vector<uint8_t>> act;  // act[l], l = 1..L
    std::vector<double> beta, q, bdata, bp_last, bm_last;
    double Z0 = 0.0;
    int64_t cum = 0, degen = 0;
    int wam_iter = 0;
    // separable 3D Haar (pin P3): act[l] is over (nz>>l, ny>>l, nx>>l) blocks
    bool haar3 = false;
    // 3D: Psi lists per (level, in-plane block) with any active z-block (and,
    // at reference precision, every level-L block for the approximation split)
    std::vector<PsiLevel> psi;                              // [l]
    // mirror mode: explicit negative-phi columns for active details, per slice-0 Mallat z
    std::vector<uint64_t> nphi_ptr;
    std::vector<uint32_t> nphi_row;
    std::vector<double> nphi_val;
    std::chrono::steady_clock::time_point t0;

    double st(double x) const { return mirror ? (double)(float)x : x; }
};

namespace orc {

static void build_matrix(orc_problem* p) {
    const Geom& g = p->g;
    const int V = g.views(), D = g.detectors;
    p->Ms = (uint64_t)V * D;
    p->Ns = (uint64_t)g.nx * g.ny;
    p->nz = g.nz;
    p->rays.resize(p->Ms);
    for (int v = 0; v < V; ++v)
        for (int k = 0; k < D; ++k) p->rays[(uint64_t)v * D + k] = make_ray(g, v, k);
    // threaded two-pass trace (count, then fill in place): each row holds the
    // entries of trace_ray in Siddon order, exactly as the serial build emits them
    int nt = resolve_threads(p->threads);
    std::vector<uint64_t> cnt(p->Ms);
    parallel_for(p->Ms, nt, [&](std::size_t lo, std::size_t hi, int) {
        for (std::size_t y = lo; y < hi; ++y) {
            uint64_t c = 0;
            trace(g, p->rays[y], [&](int, int, double) { ++c; });
            cnt[y] = c;
        }
    });
    p->rp.assign(p->Ms + 1, 0);
    for (uint64_t y = 0; y < p->Ms; ++y) p->rp[y + 1] = p->rp[y] + cnt[y];
    std::vector<uint64_t>().swap(cnt);
    const uint64_t nnz = p->rp[p->Ms];
    p->ci.resize(nnz);
    const bool f32 = p->slim && p->mirror;
    if (!p->slim) p->hexact.resize(nnz);
    if (f32) p->hv32.resize(nnz); else p->hv.resize(nnz);
    parallel_for(p->Ms, nt, [&](std::size_t lo, std::size_t hi, int) {
        for (std::size_t y = lo; y < hi; ++y) {
            uint64_t k = p->rp[y];
            trace(g, p->rays[y], [&](int ix, int iy, double len) {
                p->ci[k] = (uint32_t)iy * (uint32_t)g.nx + (uint32_t)ix;  // projector.hpp:141
                if (!p->slim) p->hexact[k] = len;
                if (f32) p->hv32[k] = (float)len; else p->hv[k] = p->st(len);
                ++k;
            });
        }
    });
    if (p->slim) return;
    // system_matrix.hpp:61-75 counting-sort transpose (rows ascending per column)
    p->cp.assign(p->Ns + 1, 0);
    for (uint32_t c : p->ci) p->cp[c + 1]++;
    for (uint64_t c = 0; c < p->Ns; ++c) p->cp[c + 1] += p->cp[c];
    p->ri.resize(nnz); p->cv.resize(nnz);
    std::vector<uint64_t> next(p->cp.begin(), p->cp.end() - 1);
    for (uint64_t y = 0; y < p->Ms; ++y)
        for (uint64_t k = p->rp[y]; k < p->rp[y + 1]; ++k) {
            uint64_t dst = next[p->ci[k]]++;
            p->ri[dst] = (uint32_t)y;
            p->cv[dst] = p->hv[k];
        }
}

// Slab transposes: a[s*n + i] <-> t[i*nz + s] (the 3D loops below keep one
// voxel's or one ray's nz values contiguous; the summation orders are those of
// the per-slice loops, so the results are bit-identical).
static void to_slab(const double* a, uint64_t n, int nz, std::vector<double>& t, int threads) {
    t.resize(n * (uint64_t)nz);
    parallel_for(n, threads, [&](std::size_t lo, std::size_t hi, int) {
        for (std::size_t i = lo; i < hi; ++i)
            for (int s = 0; s < nz; ++s) t[i * nz + s] = a[(uint64_t)s * n + i];
    });
}
static void from_slab(const std::vector<double>& t, uint64_t n, int nz, double* a, int threads) {
    parallel_for(n, threads, [&](std::size_t lo, std::size_t hi, int) {
        for (int s = 0; s < nz; ++s)
            for (std::size_t i = lo; i < hi; ++i) a[(uint64_t)s * n + i] = t[i * nz + s];
    });
}

// forward_project: l(s*M+y) = sum_k h_k mu(s*N+col_k), CSR order.
static void forward(const orc_problem* p, const double* mu, double* out) {
    if (p->nz > 1) {  // slab form: one ray's entries applied to all slices at once
        const int nz = p->nz;
        std::vector<double> muT, lT(p->Ms * (uint64_t)nz);
        to_slab(mu, p->Ns, nz, muT, p->threads);
        parallel_for(p->Ms, p->threads, [&](std::size_t lo, std::size_t hi, int) {
            std::vector<double> acc((std::size_t)nz);
            for (std::size_t y = lo; y < hi; ++y) {
                std::fill(acc.begin(), acc.end(), 0.0);
                double* a = acc.data();
                for (uint64_t k = p->rp[y]; k < p->rp[y + 1]; ++k) {
                    const double h = p->hvk(k);
                    const double* m = muT.data() + (uint64_t)p->ci[k] * nz;
                    for (int s = 0; s < nz; ++s) a[s] += h * m[s];
                }
                std::copy(acc.begin(), acc.end(), lT.begin() + y * nz);
            }
        });
        from_slab(lT, p->Ms, nz, out, p->threads);
        return;
    }
    parallel_for(p->Ms, p->threads, [&](std::size_t lo, std::size_t hi, int) {
        for (int s = 0; s < p->nz; ++s) {
            const double* m = mu + (uint64_t)s * p->Ns;
            for (std::size_t y = lo; y < hi; ++y) {
                double acc = 0.0;
                for (uint64_t k = p->rp[y]; k < p->rp[y + 1]; ++k) acc += p->hvk(k) * m[p->ci[k]];
                out[(uint64_t)s * p->Ms + y] = acc;
            }
        }
    });
}

// back_project: voxel-driven gather over the CSC mirror.
static void back(const orc_problem* p, const double* w, double* out) {
    if (p->nz > 1 || p->slim) {
        const int nz = p->nz;
        std::vector<double> wT, gT(p->Ns * (uint64_t)nz, 0.0);
        to_slab(w, p->Ms, nz, wT, p->threads);
        if (!p->slim) {  // CSC gather, rows ascending per column
            parallel_for(p->Ns, p->threads, [&](std::size_t lo, std::size_t hi, int) {
                for (std::size_t x = lo; x < hi; ++x) {
                    double* a = gT.data() + x * nz;
                    for (uint64_t k = p->cp[x]; k < p->cp[x + 1]; ++k) {
                        const double h = p->cv[k];
                        const double* ws = wT.data() + (uint64_t)p->ri[k] * nz;
                        for (int s = 0; s < nz; ++s) a[s] += h * ws[s];
                    }
                }
            });
        } else {  // CSR scatter in ascending ray order (== the CSC order), slice groups per thread
            const int G = std::min(resolve_threads(p->threads), nz);
            parallel_for((std::size_t)G, G, [&](std::size_t lo, std::size_t hi, int) {
                for (std::size_t gi = lo; gi < hi; ++gi) {
                    const int s0 = (int)((uint64_t)nz * gi / G), s1 = (int)((uint64_t)nz * (gi + 1) / G);
                    for (uint64_t y = 0; y < p->Ms; ++y) {
                        const double* ws = wT.data() + y * nz;
                        for (uint64_t k = p->rp[y]; k < p->rp[y + 1]; ++k) {
                            const double h = p->hvk(k);
                            double* a = gT.data() + (uint64_t)p->ci[k] * nz;
                            for (int s = s0; s < s1; ++s) a[s] += h * ws[s];
                        }
                    }
                }
            });
        }
        from_slab(gT, p->Ns, nz, out, p->threads);
        return;
    }
    parallel_for(p->Ns, p->threads, [&](std::size_t lo, std::size_t hi, int) {
        for (int s = 0; s < p->nz; ++s) {
            const double* ws = w + (uint64_t)s * p->Ms;
            for (std::size_t x = lo; x < hi; ++x) {
                double acc = 0.0;
                for (uint64_t k = p->cp[x]; k < p->cp[x + 1]; ++k) acc += p->cv[k] * ws[p->ri[k]];
                out[(uint64_t)s * p->Ns + x] = acc;
            }
        }
    });
}

// I-divergence term, SPEC.md:90-98 (0*ln0 = 0).
static inline double idiv_term(double d, double q) {
    return (d > 0.0 ? d * std::log(d / q) : 0.0) - d + q;
}

// ---- Haar.  One level on the leading h x w block of a slice
// (row stride nx).  Fixed operation order shared with the GPU kernels:
//   s1=a+b, s2=c+d, d1=a-b, d2=c-d; A=(s1+s2)/2 H=(s1-s2)/2 V=(d1+d2)/2 D=(d1-d2)/2
// A -> (i,j), H -> (i+h/2, j), V -> (i, j+w/2), D -> (i+h/2, j+w/2).
static void haar_fwd_level(double* x, int nx, int h, int w, std::vector<double>& tmp) {
    tmp.assign((std::size_t)h * w, 0.0);
    const int h2 = h / 2, w2 = w / 2;
    for (int i = 0; i < h2; ++i)
        for (int j = 0; j < w2; ++j) {
            double a = x[(2 * i) * nx + 2 * j], b = x[(2 * i) * nx + 2 * j + 1];
            double c = x[(2 * i + 1) * nx + 2 * j], d = x[(2 * i + 1) * nx + 2 * j + 1];
            double s1 = a + b, s2 = c + d, d1 = a - b, d2 = c - d;
            tmp[(std::size_t)i * w + j] = (s1 + s2) * 0.5;
            tmp[(std::size_t)(i + h2) * w + j] = (s1 - s2) * 0.5;
            tmp[(std::size_t)i * w + j + w2] = (d1 + d2) * 0.5;
            tmp[(std::size_t)(i + h2) * w + j + w2] = (d1 - d2) * 0.5;
        }
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < w; ++j) x[i * nx + j] = tmp[(std::size_t)i * w + j];
}
// Inverse: p=A+H m=A-H r=V+D t=V-D; a=(p+r)/2 b=(p-r)/2 c=(m+t)/2 d=(m-t)/2.
static void haar_inv_level(double* x, int nx, int h, int w, std::vector<double>& tmp) {
    tmp.assign((std::size_t)h * w, 0.0);
    const int h2 = h / 2, w2 = w / 2;
    for (int i = 0; i < h2; ++i)
        for (int j = 0; j < w2; ++j) {
            double A = x[i * nx + j], H = x[(i + h2) * nx + j];
            double Vv = x[i * nx + j + w2], Dd = x[(i + h2) * nx + j + w2];
            double pp = A + H, mm = A - H, r = Vv + Dd, t = Vv - Dd;
            tmp[(std::size_t)(2 * i) * w + 2 * j] = (pp + r) * 0.5;
            tmp[(std::size_t)(2 * i) * w + 2 * j + 1] = (pp - r) * 0.5;
            tmp[(std::size_t)(2 * i + 1) * w + 2 * j] = (mm + t) * 0.5;
            tmp[(std::size_t)(2 * i + 1) * w + 2 * j + 1] = (mm - t) * 0.5;
        }
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < w; ++j) x[i * nx + j] = tmp[(std::size_t)i * w + j];
}
static void check_haar_dims(int nx, int ny, int L) {
    if (L < 0 || L > 20) throw config_error("haar: invalid depth");
    if ((nx % (1 << L)) != 0 || (ny % (1 << L)) != 0)
        throw config_error("haar: slice dimensions not divisible by 2^L");  // SPEC.md:214, E4
}
static void dwt2(int nx, int ny, int ns, int L, const double* in, double* out) {
    check_haar_dims(nx, ny, L);
    std::vector<double> tmp;
    const std::size_t N = (std::size_t)nx * ny;
    std::copy(in, in + N * ns, out);
    for (int s = 0; s < ns; ++s)
        for (int l = 1; l <= L; ++l) haar_fwd_level(out + s * N, nx, ny >> (l - 1), nx >> (l - 1), tmp);
}
static void idwt2(int nx, int ny, int ns, int L, const double* in, double* out) {
    check_haar_dims(nx, ny, L);
    std::vector<double> tmp;
    const std::size_t N = (std::size_t)nx * ny;
    std::copy(in, in + N * ns, out);
    for (int s = 0; s < ns; ++s)
        for (int l = L; l >= 1; --l) haar_inv_level(out + s * N, nx, ny >> (l - 1), nx >> (l - 1), tmp);
}

// Mallat indices of the level-l block (bi, bj): approx only at l == L.
struct BlockIdx { uint32_t A, H, V, D; };
static inline BlockIdx mallat(int nx, int ny, int l, int bi, int bj) {
    const int hl = ny >> l, wl = nx >> l;
    BlockIdx r;
    r.A = (uint32_t)(bi * nx + bj);
    r.H = (uint32_t)((hl + bi) * nx + bj);
    r.V = (uint32_t)(bi * nx + wl + bj);
    r.D = (uint32_t)((hl + bi) * nx + wl + bj);
    return r;
}

// Per-ray walk producing phi(y|z) = sum_{x in block} h(y|x) w(x|z) for every
// block the ray crosses, at every level (SPEC.md:239-247 phi_column,
// PAPER.md:134).  A ray's cells inside a block are contiguous in Siddon order
// (cells are monotone in ix and iy), so a block is complete when the ray leaves
// it.  Summation order (fixed here, mirrored bit-for-bit by the GPU walk;
// SPEC.md:109 allows any deterministic order): a level-l block keeps four
// quadrant sums TL, TR, BL, BR, each the sequential ray-order sum of h over the
// cells of that 2^(l-1) x 2^(l-1) quadrant; on exit
//   st = TL+TR, sb = BL+BR, A = st+sb, H = st-sb, V = (TL+BL)-(TR+BR),
//   D = (TL+BR)-(TR+BL);  phi = 2^-l * (A | H | V | D)   (A only at l == L).
// Sign patterns: H + on the top half, V + on the left half, D + on TL/BR
// (Haar analysis of DESIGN.md §3).  cb(level, bi, bj, phiA, phiH, phiV, phiD)
// fires for every block in ray order within each level (phiA = 2^-l A at every
// level; the 2D model uses it at l == L, the separable 3D model at all levels).
template <typename CB>
static void phi_walk(const orc_problem* p, int L, uint64_t y, CB&& cb) {
    const int nx = p->g.nx;
    if (L == 0) {  // Omega = I: every voxel is its own approximation block
        for (uint64_t k = p->rp[y]; k < p->rp[y + 1]; ++k) {
            const int ix = (int)(p->ci[k] % (uint32_t)nx), iy = (int)(p->ci[k] / (uint32_t)nx);
            cb(0, iy, ix, p->hvk(k), 0.0, 0.0, 0.0);
        }
        return;
    }
    int cur[24], cbi[24], cbj[24];
    double q[24][4];
    for (int l = 0; l <= L; ++l) { cur[l] = -1; cbi[l] = cbj[l] = 0; q[l][0] = q[l][1] = q[l][2] = q[l][3] = 0.0; }
    auto flush = [&](int l) {
        const double TL = q[l][0], TR = q[l][1], BL = q[l][2], BR = q[l][3];
        const double st = TL + TR, sb = BL + BR;
        const double H = st - sb, V = (TL + BL) - (TR + BR), D = (TL + BR) - (TR + BL);
        const double sc = std::ldexp(1.0, -l);
        cb(l, cbi[l], cbj[l], (st + sb) * sc, H * sc, V * sc, D * sc);
        q[l][0] = q[l][1] = q[l][2] = q[l][3] = 0.0;
    };
    for (uint64_t k = p->rp[y]; k < p->rp[y + 1]; ++k) {
        const int ix = (int)(p->ci[k] % (uint32_t)nx), iy = (int)(p->ci[k] / (uint32_t)nx);
        const double h = p->hvk(k);
        for (int l = 1; l <= L; ++l) {
            const int bi = iy >> l, bj = ix >> l;
            const int key = bi * (nx >> l) + bj;
            if (key != cur[l]) {
                if (cur[l] >= 0) flush(l);
                cur[l] = key; cbi[l] = bi; cbj[l] = bj;
            }
            q[l][(((iy >> (l - 1)) & 1) << 1) | ((ix >> (l - 1)) & 1)] += h;
        }
    }
    for (int l = 1; l <= L; ++l)
        if (cur[l] >= 0) flush(l);
}

static inline bool is_active(const orc_problem* p, int l, int bi, int bj) {
    return p->act[l][(std::size_t)bi * (p->g.nx >> l) + bj] != 0;
}

// Z(y) = sum_{z in Zs} |phi(y|z)|, Eq. (1.61).
//   mirror = 0: f64, per level running sums in ray order;
//               Z = totA + tot_L + ... + tot_1.
//   mirror = 1 (== the GPU, pin P8): int64 multiples of 2^-32 with every term
//               rounded UP, Z = F(totA) + sum over active detail blocks of
//               F(|phi_H|) + F(|phi_V|) + F(|phi_D|), F(x) = ceil(x 2^32).  Exact
//               integer sums are order-independent, so the GPU keeps Z(y)
//               incrementally across expansions; rounding up keeps Z >= the
//               true sum (the majorization Eq. 1.61 needs), at most 2^-32 per
//               term above it.
static inline long long zfix_up(double x) { return (long long)std::ceil(x * 4294967296.0); }
static double z_row(const orc_problem* p, uint64_t y) {
    const int L = p->L;
    if (p->mirror) {
        double totA = 0.0;
        long long zf = 0;
        phi_walk(p, L, y, [&](int l, int bi, int bj, double pA, double pH, double pV, double pD) {
            if (l == L) totA += std::fabs(pA);
            if (l >= 1 && is_active(p, l, bi, bj))
                zf += zfix_up(std::fabs(pH)) + zfix_up(std::fabs(pV)) + zfix_up(std::fabs(pD));
        });
        return (double)(zfix_up(totA) + zf) * (1.0 / 4294967296.0);
    }
    double totA = 0.0, tot[24];
    for (int l = 0; l <= L; ++l) tot[l] = 0.0;
    phi_walk(p, L, y, [&](int l, int bi, int bj, double pA, double pH, double pV, double pD) {
        if (l == L) totA += std::fabs(pA);
        if (l >= 1 && is_active(p, l, bi, bj)) tot[l] += std::fabs(pH) + std::fabs(pV) + std::fabs(pD);
    });
    double z = totA;
    for (int l = L; l >= 1; --l) z += tot[l];
    return z;
}

static double z_row3(const orc_problem* p, uint64_t y);
static void compute_z0(orc_problem* p) {
    std::vector<double> zr(p->Ms);
    parallel_for(p->Ms, p->threads, [&](std::size_t lo, std::size_t hi, int) {
        for (std::size_t y = lo; y < hi; ++y) zr[y] = p->haar3 ? z_row3(p, y) : z_row(p, y);
    });
    double m = 0.0;
    for (double v : zr) m = std::max(m, v);
    if (!(m > 0.0)) throw numeric_error("Z0: no ray intersects the active set");
    p->Z0 = m;
}

// Explicit negative-phi columns (mirror mode, == the GPU's Phi^- CSC): for every
// active detail coefficient of slice 0, rays ascending, value (float)phi < 0.
// Ray chunks with a FIXED count (independent of the thread count), so that
// chunk-ordered combinations are deterministic on any host.
static constexpr std::size_t kRayChunks = 64;
static inline std::size_t chunk_lo(std::size_t n, std::size_t C, std::size_t c) { return n * c / C; }

// Two-pass bucket fill over rays: count(y, add) calls add(bucket) per entry;
// fill(y, put) calls put(bucket, entry) in the same order.  Entries of a
// bucket end up in ascending ray order (chunks are contiguous ray ranges and
// are laid out in chunk order) whatever the thread count.
template <typename Entry, typename Walk, typename Store>
static void bucket_rays(const orc_problem* p, std::size_t nbuckets, std::vector<uint64_t>& ptr, Walk&& walk,
                        Store&& store) {
    const std::size_t M = p->Ms, C = std::min<std::size_t>(kRayChunks, std::max<std::size_t>(M, 1));
    std::vector<std::vector<uint64_t>> start(C);   // counts, then each chunk's write cursors
    parallel_for(C, p->threads, [&](std::size_t lo, std::size_t hi, int) {
        for (std::size_t c = lo; c < hi; ++c) {
            start[c].assign(nbuckets, 0);
            for (std::size_t y = chunk_lo(M, C, c); y < chunk_lo(M, C, c + 1); ++y)
                walk(y, [&](std::size_t b, const Entry&) { start[c][b]++; });
        }
    });
    ptr.assign(nbuckets + 1, 0);
    for (std::size_t b = 0; b < nbuckets; ++b) {
        uint64_t s = ptr[b];
        for (std::size_t c = 0; c < C; ++c) { const uint64_t n = start[c][b]; start[c][b] = s; s += n; }
        ptr[b + 1] = s;
    }
    store((uint64_t)ptr[nbuckets], Entry{});   // sizing call: index == total
    parallel_for(C, p->threads, [&](std::size_t lo, std::size_t hi, int) {
        for (std::size_t c = lo; c < hi; ++c) {
            auto& st = start[c];
            for (std::size_t y = chunk_lo(M, C, c); y < chunk_lo(M, C, c + 1); ++y)
                walk(y, [&](std::size_t b, const Entry& e) { store(st[b]++, e); });
        }
    });
}

static void build_nphi(orc_problem* p) {
    const int L = p->L, nx = p->g.nx;
    const uint64_t N = p->Ns;
    using E = std::pair<uint32_t, double>;
    bool sized = false;
    auto store = [&](uint64_t i, const E& e) {
        if (!sized) { p->nphi_row.resize(i); p->nphi_val.resize(i); sized = true; return; }
        p->nphi_row[i] = e.first; p->nphi_val[i] = e.second;
    };
    bucket_rays<E>(p, N, p->nphi_ptr, [&](std::size_t y, auto&& put) {
        phi_walk(p, L, y, [&](int l, int bi, int bj, double, double pH, double pV, double pD) {
            if (l < 1 || !is_active(p, l, bi, bj)) return;
            BlockIdx z = mallat(nx, p->g.ny, l, bi, bj);
            double v[3] = {(double)(float)pH, (double)(float)pV, (double)(float)pD};
            uint32_t zz[3] = {z.H, z.V, z.D};
            for (int t = 0; t < 3; ++t)
                if (v[t] < 0.0) put(zz[t], E{(uint32_t)y, v[t]});
        });
    }, store);
}

// Direct signed split (reference mode): b+(z), b-(z) for every active z of all
// slices from the same q.  Rays are cut
// into kRayChunks fixed chunks; chunk partials are combined in chunk order (a
// wave of one chunk per thread at a time bounds the memory), so the result
// does not depend on the thread count.
static void direct_split(const orc_problem* p, const std::vector<double>& w, std::vector<double>& bp,
                         std::vector<double>& bm, bool all_coeffs) {
    const int L = p->L, nx = p->g.nx, ny = p->g.ny, nz = p->nz;
    const uint64_t N = p->Ns, M = p->Ms, NT = N * nz;
    const std::size_t C = std::min<std::size_t>(kRayChunks, std::max<uint64_t>(M, 1));
    const int nt = (int)std::min<std::size_t>((std::size_t)resolve_threads(p->threads), C);
    bp.assign(NT, 0.0); bm.assign(NT, 0.0);
    std::vector<std::vector<double>> tp(nt), tm(nt);
    for (std::size_t c0 = 0; c0 < C; c0 += nt) {
        const std::size_t nw = std::min<std::size_t>(nt, C - c0);
        parallel_for(nw, nt, [&](std::size_t wlo, std::size_t whi, int) {
          for (std::size_t wi = wlo; wi < whi; ++wi) {
            tp[wi].assign(NT, 0.0); tm[wi].assign(NT, 0.0);
            auto& P = tp[wi]; auto& Mn = tm[wi];
            const std::size_t lo = chunk_lo(M, C, c0 + wi), hi = chunk_lo(M, C, c0 + wi + 1);
        for (std::size_t y = lo; y < hi; ++y) {
            phi_walk(p, L, y, [&](int l, int bi, int bj, double pA, double pH, double pV, double pD) {
                for (int s = 0; s < nz; ++s) {
                    const double qy = w[(uint64_t)s * M + y];
                    const uint64_t off = (uint64_t)s * N;
                    if (l == 0) {  // L == 0: voxel-level approx
                        P[off + (uint64_t)bi * nx + bj] += qy * pA;
                        continue;
                    }
                    BlockIdx z = mallat(nx, ny, l, bi, bj);
                    if (l == L) {
                        double t = qy * pA;
                        if (pA > 0.0) P[off + z.A] += t; else if (pA < 0.0) Mn[off + z.A] += t;
                    }
                    if (all_coeffs || is_active(p, l, bi, bj)) {
                        double ph[3] = {pH, pV, pD};
                        uint32_t zz[3] = {z.H, z.V, z.D};
                        for (int t = 0; t < 3; ++t) {
                            double v = qy * ph[t];
                            if (ph[t] > 0.0) P[off + zz[t]] += v;
                            else if (ph[t] < 0.0) Mn[off + zz[t]] += v;
                        }
                    }
                }
            });
        }
          }
        });
        for (std::size_t wi = 0; wi < nw; ++wi)   // chunk order
            for (uint64_t z = 0; z < NT; ++z) { bp[z] += tp[wi][z]; bm[z] += tm[wi][z]; }
    }
}

// solve_coefficient_update, SPEC.md:362-370, 400, 403 with errata E1/E2:
// b+ u^2 - b u + b- = 0, u = exp(-Z0 (beta~ - beta^)), beta~ = beta^ - ln(u)/Z0.
// returns 0 updated, 1 skipped (b+ = b- = 0), 2 degenerate (no positive root).
static int solve_update(double b, double bp, double bm, double Z0, double beta, double* out) {
    *out = beta;
    if (std::fabs(bm) < 1e-300) bm = 0.0;
    if (bp == 0.0 && bm == 0.0) return 1;
    double u;
    if (bp > 0.0) {
        if (bm == 0.0) {
            if (!(b > 0.0)) return 2;
            u = b / bp;                                   // E2: u = b / b+
        } else {
            double sq = std::sqrt(b * b - 4.0 * bp * bm);
            u = (b >= 0.0) ? (b + sq) / (2.0 * bp) : (2.0 * bm) / (b - sq);  // stable form
        }
    } else {
        if (!(b < 0.0)) return 2;
        u = bm / b;
    }
    if (!(u > 0.0) || !std::isfinite(u)) return 2;
    double nb = beta - std::log(u) / Z0;
    if (!std::isfinite(nb)) throw numeric_error("wam: non-finite coefficient update");
    *out = nb;
    return 0;
}

static int64_t active_count(const orc_problem* p) {
    const int L = p->L, nx = p->g.nx, ny = p->g.ny;
    int64_t c = (int64_t)(nx >> L) * (ny >> L);
    for (int l = 1; l <= L; ++l)
        for (uint8_t a : p->act[l]) c += 3 * (int64_t)(a != 0);
    return c * p->nz;
}

// q = st(I0 exp(-H mu)) and objective I(d || q) from the unrounded q.
static double refresh_q(orc_problem* p, const std::vector<double>& mu, std::vector<double>& qout) {
    const uint64_t MT = p->Ms * p->nz;
    std::vector<double> l(MT), term(MT);
    forward(p, mu.data(), l.data());
    qout.resize(MT);
    parallel_for(MT, p->threads, [&](std::size_t lo, std::size_t hi, int) {
        for (std::size_t y = lo; y < hi; ++y) {
            if (!std::isfinite(l[y])) throw numeric_error("non-finite line integral at ray " + std::to_string(y));
            double qq = p->I0[y] * std::exp(-l[y]);
            term[y] = idiv_term(p->d[y], qq);
            qout[y] = p->st(qq);
        }
    });
    double obj = 0.0;
    for (uint64_t y = 0; y < MT; ++y) obj += term[y];
    return obj;
}

static void set_data(orc_problem* p, const double* d, const double* I0) {
    const uint64_t MT = p->Ms * p->nz;
    p->d.resize(MT); p->I0.resize(MT);
    for (uint64_t y = 0; y < MT; ++y) {
        if (!(d[y] >= 0.0)) throw contract_error("data: d must be >= 0");
        if (!(I0[y] > 0.0)) throw contract_error("data: I0 must be > 0");
        p->d[y] = p->st(d[y]);
        p->I0[y] = p->st(I0[y]);
    }
}

static void idwt3(int nx, int ny, int nz, int L, const double* in, double* out);
static std::vector<double> image_of_beta(const orc_problem* p, bool round_storage) {
    std::vector<double> mu(p->beta.size());
    if (p->haar3) idwt3(p->g.nx, p->g.ny, p->g.nz, p->L, p->beta.data(), mu.data());
    else idwt2(p->g.nx, p->g.ny, p->nz, p->L, p->beta.data(), mu.data());
    if (round_storage)
        for (auto& v : mu) v = p->st(v);
    return mu;
}


// ======================================================================
// Separable 3D Haar (pin P3): the same 1D orthonormal step
// along z on top of the in-plane 2D step.  One level on the leading
// d x h x w region of the volume (z-major, row stride nx, plane stride N):
// each z-plane pair (2k, 2k+1) gets the in-plane 2D step (DESIGN.md §3 order)
// giving (A,H,V,D)_0 and (A,H,V,D)_1, then low = (P0+P1)*c, high = (P0-P1)*c
// with c = 1/sqrt(2) rounded to double.  Mallat positions: low at plane k,
// high at plane k + d/2; in-plane positions as in 2D.
static constexpr double kC3 = 0.70710678118654752440;

static inline double cpow3(int l) {  // c^l by repeated multiplication (GPU mirrors this)
    double c = 1.0;
    for (int i = 0; i < l; ++i) c *= kC3;
    return c;
}

static void haar3_fwd_level(double* x, int nx, int N, int d, int h, int w, std::vector<double>& tmp) {
    tmp.assign((std::size_t)d * h * w, 0.0);
    const int d2 = d / 2, h2 = h / 2, w2 = w / 2;
    auto at = [&](int z, int i, int j) -> double& { return x[(std::size_t)z * N + (std::size_t)i * nx + j]; };
    auto tt = [&](int z, int i, int j) -> double& { return tmp[((std::size_t)z * h + i) * w + j]; };
    for (int k = 0; k < d2; ++k)
        for (int i = 0; i < h2; ++i)
            for (int j = 0; j < w2; ++j) {
                double P[2][4];
                for (int e = 0; e < 2; ++e) {
                    const int z = 2 * k + e;
                    const double a = at(z, 2 * i, 2 * j), b = at(z, 2 * i, 2 * j + 1);
                    const double c = at(z, 2 * i + 1, 2 * j), dd = at(z, 2 * i + 1, 2 * j + 1);
                    const double s1 = a + b, s2 = c + dd, d1 = a - b, d2v = c - dd;
                    P[e][0] = (s1 + s2) * 0.5; P[e][1] = (s1 - s2) * 0.5;
                    P[e][2] = (d1 + d2v) * 0.5; P[e][3] = (d1 - d2v) * 0.5;
                }
                const int pi[4] = {i, i + h2, i, i + h2}, pj[4] = {j, j, j + w2, j + w2};
                for (int t = 0; t < 4; ++t) {
                    tt(k, pi[t], pj[t]) = (P[0][t] + P[1][t]) * kC3;
                    tt(k + d2, pi[t], pj[t]) = (P[0][t] - P[1][t]) * kC3;
                }
            }
    for (int z = 0; z < d; ++z)
        for (int i = 0; i < h; ++i)
            for (int j = 0; j < w; ++j) at(z, i, j) = tt(z, i, j);
}

static void haar3_inv_level(double* x, int nx, int N, int d, int h, int w, std::vector<double>& tmp) {
    tmp.assign((std::size_t)d * h * w, 0.0);
    const int d2 = d / 2, h2 = h / 2, w2 = w / 2;
    auto at = [&](int z, int i, int j) -> double& { return x[(std::size_t)z * N + (std::size_t)i * nx + j]; };
    auto tt = [&](int z, int i, int j) -> double& { return tmp[((std::size_t)z * h + i) * w + j]; };
    for (int k = 0; k < d2; ++k)
        for (int i = 0; i < h2; ++i)
            for (int j = 0; j < w2; ++j) {
                const int pi[4] = {i, i + h2, i, i + h2}, pj[4] = {j, j, j + w2, j + w2};
                double P[2][4];
                for (int t = 0; t < 4; ++t) {
                    const double lo = at(k, pi[t], pj[t]), hi = at(k + d2, pi[t], pj[t]);
                    P[0][t] = (lo + hi) * kC3;
                    P[1][t] = (lo - hi) * kC3;
                }
                for (int e = 0; e < 2; ++e) {
                    const int z = 2 * k + e;
                    const double A = P[e][0], H = P[e][1], V = P[e][2], D = P[e][3];
                    const double pp = A + H, mm = A - H, r = V + D, t2 = V - D;
                    tt(z, 2 * i, 2 * j) = (pp + r) * 0.5;
                    tt(z, 2 * i, 2 * j + 1) = (pp - r) * 0.5;
                    tt(z, 2 * i + 1, 2 * j) = (mm + t2) * 0.5;
                    tt(z, 2 * i + 1, 2 * j + 1) = (mm - t2) * 0.5;
                }
            }
    for (int z = 0; z < d; ++z)
        for (int i = 0; i < h; ++i)
            for (int j = 0; j < w; ++j) at(z, i, j) = tt(z, i, j);
}

static void check_haar3_dims(int nx, int ny, int nz, int L) {
    check_haar_dims(nx, ny, L);
    if ((nz % (1 << L)) != 0) throw config_error("haar3: nz not divisible by 2^L");
}
static void dwt3(int nx, int ny, int nz, int L, const double* in, double* out) {
    check_haar3_dims(nx, ny, nz, L);
    const std::size_t N = (std::size_t)nx * ny;
    std::copy(in, in + N * nz, out);
    std::vector<double> tmp;
    for (int l = 1; l <= L; ++l) haar3_fwd_level(out, nx, (int)N, nz >> (l - 1), ny >> (l - 1), nx >> (l - 1), tmp);
}
static void idwt3(int nx, int ny, int nz, int L, const double* in, double* out) {
    check_haar3_dims(nx, ny, nz, L);
    const std::size_t N = (std::size_t)nx * ny;
    std::copy(in, in + N * nz, out);
    std::vector<double> tmp;
    for (int l = L; l >= 1; --l) haar3_inv_level(out, nx, (int)N, nz >> (l - 1), ny >> (l - 1), nx >> (l - 1), tmp);
}

// 3D Mallat indices of level-l block (bk, bi, bj): [0] approx (l == L), then the
// 7 details in the fixed order Hl, Vl, Dl, Ah, Hh, Vh, Dh (l = z low / h = z high).
static inline void mallat3(int nx, int ny, int nz, int l, int bk, int bi, int bj, uint64_t (&z)[8]) {
    const uint64_t N = (uint64_t)nx * ny;
    const int dl = nz >> l, hl = ny >> l, wl = nx >> l;
    auto ix3 = [&](int zz, int yy, int xx) { return (uint64_t)zz * N + (uint64_t)yy * nx + xx; };
    z[0] = ix3(bk, bi, bj);
    z[1] = ix3(bk, hl + bi, bj); z[2] = ix3(bk, bi, wl + bj); z[3] = ix3(bk, hl + bi, wl + bj);
    z[4] = ix3(dl + bk, bi, bj); z[5] = ix3(dl + bk, hl + bi, bj); z[6] = ix3(dl + bk, bi, wl + bj);
    z[7] = ix3(dl + bk, hl + bi, wl + bj);
}
static inline std::size_t blk3(const orc_problem* p, int l, int bk, int bi, int bj) {
    return ((std::size_t)bk * (p->g.ny >> l) + bi) * (p->g.nx >> l) + bj;
}
static inline bool active3(const orc_problem* p, int l, int bk, int bi, int bj) {
    return p->act[l][blk3(p, l, bk, bi, bj)] != 0;
}

// Z(y, s) = zA(y) + tot_L(y, k_L(s)) + ... + tot_1(y, k_1(s)) with
//   zA = sum over level-L in-plane blocks (ray order) of |psi_A c^L|,
//   tot_l(y, k) = sum over level-l in-plane blocks b (ray order) with (k, b)
//   active of t(b) = |Hl|+|Vl|+|Dl|+|Ah|+|Hh|+|Vh|+|Dh| (that order, each psi c^l).
// Returns max_s Z(y, s) (Eq. 1.61 over the rays of every slice).
static double z_row3(const orc_problem* p, uint64_t y) {
    const int L = p->L, nz = p->g.nz;
    double zA = 0.0;
    static thread_local std::vector<std::vector<double>> tot;
    tot.resize(L + 1);
    for (int l = 1; l <= L; ++l) tot[l].assign(nz >> l, 0.0);
    const double cL = cpow3(L);
    phi_walk(p, L, y, [&](int l, int bi, int bj, double pA, double pH, double pV, double pD) {
        const double cl = cpow3(l);
        if (l == L) zA += std::fabs(pA * cL);
        const double h = std::fabs(pH * cl), v = std::fabs(pV * cl), dd = std::fabs(pD * cl), a = std::fabs(pA * cl);
        const double t = (((((h + v) + dd) + a) + h) + v) + dd;
        for (int k = 0; k < (nz >> l); ++k)
            if (active3(p, l, k, bi, bj)) tot[l][k] += t;
    });
    double best = 0.0;
    for (int s = 0; s < nz; ++s) {
        double z = zA;
        for (int l = L; l >= 1; --l) z += tot[l][s >> l];
        best = std::max(best, z);
    }
    return best;
}

// Psi lists of level l over the in-plane blocks with want[b] != 0: rays
// ascending, (psi_A, psi_H, psi_V, psi_D) fp32-rounded in mirror mode.
static void build_psi_level(const orc_problem* p, int l, const std::vector<uint8_t>& want, PsiLevel& out) {
    const int L = p->L, nx = p->g.nx;
    const int wl = nx >> l;
    const bool r32 = p->mirror;
    struct E { uint32_t y; std::array<double, 4> v; };
    bool sized = false;
    auto store = [&](uint64_t i, const E& e) {
        if (!sized) { out.ray.resize(i); out.val.resize(i); sized = true; return; }
        out.ray[i] = e.y; out.val[i] = e.v;
    };
    bucket_rays<E>(p, want.size(), out.ptr, [&](std::size_t y, auto&& put) {
        phi_walk(p, L, y, [&](int ll, int bi, int bj, double pA, double pH, double pV, double pD) {
            if (ll != l) return;
            const std::size_t b = (std::size_t)bi * wl + bj;
            if (!want[b]) return;
            if (r32) put(b, E{(uint32_t)y, {(double)(float)pA, (double)(float)pH, (double)(float)pV, (double)(float)pD}});
            else put(b, E{(uint32_t)y, {pA, pH, pV, pD}});
        });
    }, store);
}

// in-plane blocks of level l with any active z-block (all of them at level L
// when the approximations are split directly, i.e. at reference precision)
static std::vector<uint8_t> psi_want(const orc_problem* p, int l, bool all) {
    const int nx = p->g.nx, ny = p->g.ny, nz = p->g.nz;
    const int hl = ny >> l, wl = nx >> l;
    std::vector<uint8_t> w((std::size_t)hl * wl, all ? 1 : 0);
    if (!all)
        for (int k = 0; k < (nz >> l); ++k)
            for (std::size_t b = 0; b < w.size(); ++b)
                if (p->act[l][(std::size_t)k * w.size() + b]) w[b] = 1;
    return w;
}

static void build_psi3(orc_problem* p) {
    const int L = p->L;
    p->psi.assign(L + 1, {});
    for (int l = 1; l <= L; ++l) build_psi_level(p, l, psi_want(p, l, !p->mirror && l == L), p->psi[l]);
}

// b-(z) of every active 3D detail (mirror mode, from the Psi lists):
//   z-low  subband p: sum_y [psi_p < 0] psi_p c^l (Qlo + Qhi)
//   z-high subband p: sum_y psi_p < 0 ? psi_p c^l Qlo : (psi_p > 0 ? -psi_p c^l Qhi : 0)
// with Qlo / Qhi the ray-wise sums of q over the lower / upper half of the
// z-block's slices (ascending slice order).  Rays ascending within a list.
// qT: q in slab layout [y][s].  Blocks are independent (parallel over them).
static void split3_mirror(const orc_problem* p, const std::vector<double>& qT, std::vector<double>& bm) {
    const int L = p->L, nx = p->g.nx, ny = p->g.ny, nz = p->g.nz;
    bm.assign(p->Ns * nz, 0.0);
    for (int l = 1; l <= L; ++l) {
        const double cl = cpow3(l);
        const int hw = 1 << (l - 1), wl = nx >> l;
        const PsiLevel& ps = p->psi[l];
        parallel_for((std::size_t)(ny >> l) * wl, p->threads, [&](std::size_t lo, std::size_t hi, int) {
            for (std::size_t b = lo; b < hi; ++b) {
                const int bi = (int)(b / wl), bj = (int)(b % wl);
                for (int k = 0; k < (nz >> l); ++k) {
                    if (!active3(p, l, k, bi, bj)) continue;
                    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
                    for (uint64_t e = ps.ptr[b]; e < ps.ptr[b + 1]; ++e) {
                        const double* qy = qT.data() + (uint64_t)ps.ray[e] * nz + (uint64_t)k * 2 * hw;
                        const auto& v = ps.val[e];
                        double qlo = 0.0, qhi = 0.0;
                        for (int s = 0; s < hw; ++s) qlo += qy[s];
                        for (int s = 0; s < hw; ++s) qhi += qy[hw + s];
                        const double qall = qlo + qhi;
                        const double A = v[0] * cl, H = v[1] * cl, V = v[2] * cl, D = v[3] * cl;
                        const double lowp[3] = {H, V, D}, highp[4] = {A, H, V, D};
                        for (int t = 0; t < 3; ++t)
                            if (lowp[t] < 0.0) acc[t] += lowp[t] * qall;
                        for (int t = 0; t < 4; ++t) {
                            if (highp[t] < 0.0) acc[3 + t] += highp[t] * qlo;
                            else if (highp[t] > 0.0) acc[3 + t] += -highp[t] * qhi;
                        }
                    }
                    uint64_t z[8];
                    mallat3(nx, ny, nz, l, k, bi, bj, z);
                    for (int t = 0; t < 7; ++t) bm[z[1 + t]] = acc[t];
                }
            }
        });
    }
}

// Direct signed split (reference precision, 3D): b+ / b- for every active z
// (or every z with all_coeffs) from the exact phi(y_s|z) = psi c^l sigma_z(s).
// Block-driven over the f64 Psi lists: every z accumulates its (ray, slice)
// terms in ascending (ray, slice) order, the order of a serial ray walk.
// all_coeffs (init): the lists of every block are built one level at a time.
static void direct_split3(const orc_problem* p, const std::vector<double>& qT, std::vector<double>& bp,
                          std::vector<double>& bm, bool all_coeffs) {
    const int L = p->L, nx = p->g.nx, ny = p->g.ny, nz = p->g.nz;
    const uint64_t NT = p->Ns * nz;
    bp.assign(NT, 0.0); bm.assign(NT, 0.0);
    const double cL = cpow3(L);
    for (int l = 1; l <= L; ++l) {
        PsiLevel tmp;
        const PsiLevel* ps = &p->psi[l];
        if (all_coeffs) { build_psi_level(p, l, psi_want(p, l, true), tmp); ps = &tmp; }
        const double cl = cpow3(l);
        const int wl = nx >> l, bz = 1 << l;
        parallel_for((std::size_t)(ny >> l) * wl, p->threads, [&](std::size_t lo, std::size_t hi, int) {
            for (std::size_t b = lo; b < hi; ++b) {
                const int bi = (int)(b / wl), bj = (int)(b % wl);
                for (int k = 0; k < (nz >> l); ++k) {
                    const bool act = all_coeffs || active3(p, l, k, bi, bj), doA = l == L;
                    if (!act && !doA) continue;
                    double P[8] = {0, 0, 0, 0, 0, 0, 0, 0}, Mn[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    auto add = [&](int t, double v, double phi) {
                        if (phi > 0.0) P[t] += v; else if (phi < 0.0) Mn[t] += v;
                    };
                    for (uint64_t e = ps->ptr[b]; e < ps->ptr[b + 1]; ++e) {
                        const double* qy = qT.data() + (uint64_t)ps->ray[e] * nz;
                        const double pA = ps->val[e][0], pH = ps->val[e][1], pV = ps->val[e][2], pD = ps->val[e][3];
                        for (int s = k * bz; s < (k + 1) * bz; ++s) {
                            const double q = qy[s];
                            const double sg = ((s >> (l - 1)) & 1) ? -1.0 : 1.0;
                            if (doA) { const double ph = pA * cL; add(0, q * ph, ph); }
                            if (!act) continue;
                            const double ph[7] = {pH * cl, pV * cl, pD * cl, pA * cl * sg, pH * cl * sg,
                                                  pV * cl * sg, pD * cl * sg};
                            for (int t = 0; t < 7; ++t) add(1 + t, q * ph[t], ph[t]);
                        }
                    }
                    uint64_t z[8];
                    mallat3(nx, ny, nz, l, k, bi, bj, z);
                    if (doA) { bp[z[0]] = P[0]; bm[z[0]] = Mn[0]; }
                    if (act)
                        for (int t = 1; t < 8; ++t) { bp[z[t]] = P[t]; bm[z[t]] = Mn[t]; }
                }
            }
        });
    }
}

static int64_t active_count3(const orc_problem* p) {
    const int L = p->L, nx = p->g.nx, ny = p->g.ny, nz = p->g.nz;
    int64_t c = (int64_t)(nx >> L) * (ny >> L) * (nz >> L);
    for (int l = 1; l <= L; ++l)
        for (uint8_t a : p->act[l]) c += 7 * (int64_t)(a != 0);
    return c;
}

}  // namespace orc

#define ORC_TRY(...)                                       \
    try { __VA_ARGS__; return ORC_OK; }                     \
    catch (const orc::Error& e) { g_err = e.what(); return e.code; } \
    catch (const std::exception& e) { g_err = e.what(); return ORC_ERR_CONTRACT; }

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_create_ex(const orc_geometry* gc, int mirror, int threads, int flags, orc_problem** out) {
    ORC_TRY({
        if (!out) throw contract_error("null out");
        auto* p = new orc_problem();
        try {
            p->g = make_geom(gc);
            p->mirror = mirror != 0;
            p->slim = (flags & ORC_SLIM) != 0;
            p->threads = threads;
            build_matrix(p);
        } catch (...) { delete p; throw; }
        *out = p;
    })
}

int orc_create(const orc_geometry* gc, int mirror, int threads, orc_problem** out) {
    return orc_create_ex(gc, mirror, threads, 0, out);
}

int orc_create_csr(uint64_t M, int nx, int ny, const uint64_t* rp, const uint32_t* ci, const double* val,
                   int mirror, int threads, orc_problem** out) {
    ORC_TRY({
        if (!out || !rp) throw contract_error("null argument");
        if (nx < 1 || ny < 1) throw contract_error("grid must be positive");
        auto* p = new orc_problem();
        p->g.nx = nx; p->g.ny = ny; p->g.nz = 1; p->g.detectors = 1; p->g.angles.assign(1, 0.0);
        p->mirror = mirror != 0; p->threads = threads;
        p->Ms = M; p->Ns = (uint64_t)nx * ny; p->nz = 1;
        const uint64_t nnz = rp[M];
        p->rp.assign(rp, rp + M + 1);
        p->ci.assign(ci, ci + nnz);
        p->hexact.assign(val, val + nnz);
        for (uint64_t k = 0; k < nnz; ++k)
            if (p->ci[k] >= p->Ns) { delete p; throw contract_error("column index out of range"); }
        p->hv.resize(nnz);
        for (uint64_t k = 0; k < nnz; ++k) p->hv[k] = p->st(p->hexact[k]);
        p->cp.assign(p->Ns + 1, 0);
        for (uint32_t c : p->ci) p->cp[c + 1]++;
        for (uint64_t c = 0; c < p->Ns; ++c) p->cp[c + 1] += p->cp[c];
        p->ri.resize(nnz); p->cv.resize(nnz);
        std::vector<uint64_t> next(p->cp.begin(), p->cp.end() - 1);
        for (uint64_t y = 0; y < M; ++y)
            for (uint64_t k = p->rp[y]; k < p->rp[y + 1]; ++k) {
                uint64_t dst = next[p->ci[k]]++;
                p->ri[dst] = (uint32_t)y;
                p->cv[dst] = p->hv[k];
            }
        *out = p;
    })
}

int orc_am_set_clamp(orc_problem* p, int clamp) { ORC_TRY({ p->am_clamp = clamp != 0; }) }

void orc_destroy(orc_problem* p) { delete p; }

int orc_dims(const orc_problem* p, uint64_t* M, uint64_t* N, uint64_t* nnz, int* nz) {
    ORC_TRY({
        if (M) *M = p->Ms;
        if (N) *N = p->Ns;
        if (nnz) *nnz = p->rp.back();
        if (nz) *nz = p->nz;
    })
}

int orc_get_csr(const orc_problem* p, uint64_t* rp, uint32_t* ci, double* val) {
    ORC_TRY({
        if (rp) std::copy(p->rp.begin(), p->rp.end(), rp);
        if (ci) std::copy(p->ci.begin(), p->ci.end(), ci);
        if (p->slim && (ci || val)) throw contract_error("slim problem: the exact CSR is not kept");
        if (val) std::copy(p->hexact.begin(), p->hexact.end(), val);
    })
}

int orc_get_csc(const orc_problem* p, uint64_t* cp, uint32_t* ri, double* val) {
    ORC_TRY({
        if (p->slim) throw contract_error("slim problem: no CSC mirror");
        if (cp) std::copy(p->cp.begin(), p->cp.end(), cp);
        if (ri) std::copy(p->ri.begin(), p->ri.end(), ri);
        if (val) std::copy(p->cv.begin(), p->cv.end(), val);
    })
}

int orc_get_rays(const orc_problem* p, double* r6) {
    ORC_TRY({
        for (uint64_t y = 0; y < p->Ms; ++y) {
            const Ray& r = p->rays[y];
            double* o = r6 + 6 * y;
            o[0] = r.ox; o[1] = r.oy; o[2] = r.dx; o[3] = r.dy; o[4] = r.tmin; o[5] = r.tmax;
        }
    })
}

int orc_forward_project(const orc_problem* p, const double* mu, double* out) {
    ORC_TRY({ forward(p, mu, out); })
}
int orc_back_project(const orc_problem* p, const double* w, double* out) {
    ORC_TRY({ back(p, w, out); })
}

int orc_predicted_means(uint64_t n, const double* I0, const double* l, double* q) {
    ORC_TRY({
        for (uint64_t y = 0; y < n; ++y) {
            if (!std::isfinite(l[y])) throw numeric_error("predicted_means: non-finite line integral at ray " + std::to_string(y));
            q[y] = I0[y] * std::exp(-l[y]);
        }
    })
}

int orc_i_divergence(uint64_t n, const double* d, const double* q, double* out) {
    ORC_TRY({
        double s = 0.0;
        for (uint64_t y = 0; y < n; ++y) {
            if (!(q[y] > 0.0)) throw numeric_error("i_divergence: q <= 0 at ray " + std::to_string(y));
            s += idiv_term(d[y], q[y]);
        }
        *out = s;
    })
}

int orc_rasterize(const orc_geometry* gc, const orc_primitive* pr, int np, double bg, double* mu) {
    ORC_TRY({
        Geom g = make_geom(gc);
        const double h = g.voxel;
        const double x0 = -0.5 * g.width(), y0 = -0.5 * g.height(), z0 = -0.5 * (g.nz * h);
        for (int iz = 0; iz < g.nz; ++iz)
            for (int iy = 0; iy < g.ny; ++iy)
                for (int ix = 0; ix < g.nx; ++ix) {
                    const double x = x0 + (ix + 0.5) * h, y = y0 + (iy + 0.5) * h, z = z0 + (iz + 0.5) * h;
                    double v = bg;
                    for (int i = 0; i < np; ++i) {  // painter's order
                        const orc_primitive& q = pr[i];
                        const double c = std::cos(q.angle), s = std::sin(q.angle);
                        const double dx = x - q.cx, dy = y - q.cy;
                        const double u = c * dx + s * dy, w = -s * dx + c * dy;
                        const double t = z - q.cz;
                        bool in;
                        if (q.kind == 0) {
                            double r = (u / q.ax) * (u / q.ax) + (w / q.ay) * (w / q.ay);
                            if (g.nz > 1) r += (t / q.az) * (t / q.az);
                            in = r <= 1.0;
                        } else {
                            in = std::fabs(u) <= q.ax && std::fabs(w) <= q.ay;
                            if (g.nz > 1) in = in && std::fabs(t) <= q.az;
                        }
                        if (in) v = q.value;
                    }
                    mu[((std::size_t)iz * g.ny + iy) * g.nx + ix] = v;
                }
    })
}

int orc_simulate(const orc_problem* p, const double* mu, const double* I0, uint64_t seed, int noisy,
                 double* dout) {
    ORC_TRY({
        const uint64_t M = p->Ms, N = p->Ns;
        if (!p->hexact.empty()) {
            parallel_for(M, p->threads, [&](std::size_t lo, std::size_t hi, int) {
                for (int s = 0; s < p->nz; ++s)
                    for (std::size_t y = lo; y < hi; ++y) {
                        double acc = 0.0;  // exact f64 h, CSR order
                        for (uint64_t k = p->rp[y]; k < p->rp[y + 1]; ++k)
                            acc += p->hexact[k] * mu[(uint64_t)s * N + p->ci[k]];
                        const uint64_t id = (uint64_t)s * M + y;
                        double m = I0[id] * std::exp(-acc);
                        dout[id] = noisy ? poisson(seed, id, m) : m;
                    }
            });
        } else {  // slim: exact h re-traced (the same trace_ray entries, same CSR order)
            parallel_for(M, p->threads, [&](std::size_t lo, std::size_t hi, int) {
                std::vector<std::pair<uint32_t, double>> row;
                for (std::size_t y = lo; y < hi; ++y) {
                    row.clear();
                    trace(p->g, p->rays[y], [&](int ix, int iy, double len) {
                        row.push_back({(uint32_t)iy * (uint32_t)p->g.nx + (uint32_t)ix, len});
                    });
                    for (int s = 0; s < p->nz; ++s) {
                        double acc = 0.0;
                        for (const auto& e : row) acc += e.second * mu[(uint64_t)s * N + e.first];
                        const uint64_t id = (uint64_t)s * M + y;
                        double m = I0[id] * std::exp(-acc);
                        dout[id] = noisy ? poisson(seed, id, m) : m;
                    }
                }
            });
        }
    })
}

double orc_uniform(uint64_t seed, uint64_t stream, uint64_t k) { return uniform(seed, stream, k); }
double orc_poisson(uint64_t seed, uint64_t stream, double mean) {
    try { return poisson(seed, stream, mean); } catch (...) { return -1.0; }
}

int orc_dwt2(int nx, int ny, int ns, int L, const double* in, double* out) {
    ORC_TRY({ dwt2(nx, ny, ns, L, in, out); })
}
int orc_idwt2(int nx, int ny, int ns, int L, const double* in, double* out) {
    ORC_TRY({ idwt2(nx, ny, ns, L, in, out); })
}

int orc_dwt3(int nx, int ny, int nz, int L, const double* in, double* out) {
    ORC_TRY({ dwt3(nx, ny, nz, L, in, out); })
}
int orc_idwt3(int nx, int ny, int nz, int L, const double* in, double* out) {
    ORC_TRY({ idwt3(nx, ny, nz, L, in, out); })
}

int orc_solve_update(double b, double bp, double bm, double Z0, double beta, double* out) {
    try { return solve_update(b, bp, bm, Z0, beta, out); }
    catch (const orc::Error& e) { g_err = e.what(); return -e.code; }
}

// ---------------- am-baseline, SPEC.md:292-318 ----------------
int orc_am_init(orc_problem* p, const double* d, const double* I0, const double* init_mu) {
    ORC_TRY({
        set_data(p, d, I0);
        const uint64_t NT = p->Ns * p->nz;
        p->am_mu.assign(NT, 0.0);
        if (init_mu)
            for (uint64_t x = 0; x < NT; ++x) p->am_mu[x] = p->st(init_mu[x]);
        p->am_b.resize(NT);
        back(p, p->d.data(), p->am_b.data());           // b(x) = sum_y d h
        double z0 = 0.0;                                  // Z0 = max_y sum_x h
        for (uint64_t y = 0; y < p->Ms; ++y) {
            double s = 0.0;
            for (uint64_t k = p->rp[y]; k < p->rp[y + 1]; ++k) s += p->hvk(k);
            z0 = std::max(z0, s);
        }
        if (!(z0 > 0.0)) throw numeric_error("am: Z0 must be positive");
        p->am_Z0 = z0;
        refresh_q(p, p->am_mu, p->am_q);
        p->am_iter = 0;
        p->am_ready = true;
        p->t0 = std::chrono::steady_clock::now();
    })
}

int orc_am_iterate(orc_problem* p, int n, orc_record* recs) {
    ORC_TRY({
        if (!p->am_ready) throw contract_error("am: not initialised");
        const uint64_t NT = p->Ns * p->nz;
        std::vector<double> bh(NT);
        for (int it = 0; it < n; ++it) {
            back(p, p->am_q.data(), bh.data());          // b^(x) = sum_y q^ h
            for (uint64_t x = 0; x < NT; ++x) {
                const double b = p->am_b[x], c = bh[x];
                if (!(b > 0.0) || !(c > 0.0)) continue;  // frozen voxel
                double v = p->am_mu[x] + std::log(c / b) / p->am_Z0;
                if (!std::isfinite(v)) throw numeric_error("am: non-finite update at voxel " + std::to_string(x));
                p->am_mu[x] = p->st(p->am_clamp ? std::max(0.0, v) : v);
            }
            double obj = refresh_q(p, p->am_mu, p->am_q);
            p->am_iter++;
            if (recs) {
                recs[it].iter = p->am_iter;
                recs[it].objective = obj;
                recs[it].elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - p->t0).count();
                recs[it].active_set = (int64_t)NT;
                recs[it].cum_updates = (int64_t)NT * p->am_iter;
            }
        }
    })
}

int orc_am_get(const orc_problem* p, double* mu, double* q, double* Z0, double* b) {
    ORC_TRY({
        if (mu) std::copy(p->am_mu.begin(), p->am_mu.end(), mu);
        if (q) std::copy(p->am_q.begin(), p->am_q.end(), q);
        if (Z0) *Z0 = p->am_Z0;
        if (b) std::copy(p->am_b.begin(), p->am_b.end(), b);
    })
}

// ---------------- wavelet-am, SPEC.md:353-389 ----------------
int orc_set_haar_dim(orc_problem* p, int dim) {
    ORC_TRY({
        if (dim != 2 && dim != 3) throw config_error("haar: dimension must be 2 or 3");
        p->haar3 = dim == 3;
        p->wam_ready = false;
    })
}

int orc_wam_init(orc_problem* p, const double* d, const double* I0, int L, const double* init_beta) {
    ORC_TRY({
        if (p->haar3) check_haar3_dims(p->g.nx, p->g.ny, p->g.nz, L);
        else check_haar_dims(p->g.nx, p->g.ny, L);
        set_data(p, d, I0);
        p->L = L;
        const uint64_t NT = p->Ns * p->nz;
        p->act.assign(L + 1, {});
        for (int l = 1; l <= L; ++l)
            p->act[l].assign((std::size_t)(p->g.nx >> l) * (p->g.ny >> l) * (p->haar3 ? (p->g.nz >> l) : 1), 0);
        p->beta.assign(NT, 0.0);
        if (init_beta)
            for (uint64_t z = 0; z < NT; ++z) p->beta[z] = p->st(init_beta[z]);
        // b(z) = sum_y d(y) phi(y|z) for every z (data-only)
        if (p->mirror) {
            std::vector<double> g(NT);
            back(p, p->d.data(), g.data());
            p->bdata.resize(NT);
            if (p->haar3) { dwt3(p->g.nx, p->g.ny, p->g.nz, L, g.data(), p->bdata.data()); build_psi3(p); }
            else { dwt2(p->g.nx, p->g.ny, p->nz, L, g.data(), p->bdata.data()); build_nphi(p); }
        } else {
            std::vector<double> bp, bm;
            if (p->haar3) {
                std::vector<double> dT;
                to_slab(p->d.data(), p->Ms, p->nz, dT, p->threads);
                direct_split3(p, dT, bp, bm, true);
                build_psi3(p);
            } else {
                direct_split(p, p->d, bp, bm, true);
            }
            p->bdata.resize(NT);
            for (uint64_t z = 0; z < NT; ++z) p->bdata[z] = bp[z] + bm[z];
        }
        compute_z0(p);
        std::vector<double> mu = image_of_beta(p, true);
        refresh_q(p, mu, p->q);
        p->cum = 0; p->degen = 0; p->wam_iter = 0;
        p->bp_last.assign(NT, 0.0); p->bm_last.assign(NT, 0.0);
        p->wam_ready = true;
        p->t0 = std::chrono::steady_clock::now();
    })
}

int orc_wam_iterate(orc_problem* p, int n, orc_record* recs) {
    ORC_TRY({
        if (!p->wam_ready) throw contract_error("wam: not initialised");
        const int L = p->L, nx = p->g.nx, ny = p->g.ny, nz = p->g.nz;
        const uint64_t N = p->Ns, NT = N * p->nz;
        for (int it = 0; it < n; ++it) {
            std::vector<double> bp, bm;
            if (p->mirror) {
                std::vector<double> g(NT), S(NT);
                back(p, p->q.data(), g.data());
                if (p->haar3) {
                    dwt3(nx, ny, nz, L, g.data(), S.data());
                    std::vector<double> qT;
                    to_slab(p->q.data(), p->Ms, nz, qT, p->threads);
                    split3_mirror(p, qT, bm);
                } else {
                    dwt2(nx, ny, p->nz, L, g.data(), S.data());
                    bm.assign(NT, 0.0);
                    // b-(z): exact fixed-point sum (2^-20 units) of q*phi over the
                    // Phi^- column -- order-independent, mirrored bit-for-bit by
                    // the GPU split whatever order its columns hold
                    parallel_for(N, p->threads, [&](std::size_t lo, std::size_t hi, int) {
                        for (int s = 0; s < p->nz; ++s)
                            for (uint64_t z = lo; z < hi; ++z) {
                                long long acc = 0;
                                for (uint64_t k = p->nphi_ptr[z]; k < p->nphi_ptr[z + 1]; ++k)
                                    acc += std::llrint(p->q[(uint64_t)s * p->Ms + p->nphi_row[k]] * p->nphi_val[k] *
                                                       1048576.0);
                                bm[(uint64_t)s * N + z] = (double)acc * (1.0 / 1048576.0);
                            }
                    });
                }
                bp.resize(NT);
                for (uint64_t z = 0; z < NT; ++z) bp[z] = S[z] - bm[z];
            } else if (p->haar3) {
                std::vector<double> qT;
                to_slab(p->q.data(), p->Ms, nz, qT, p->threads);
                direct_split3(p, qT, bp, bm, false);
            } else {
                direct_split(p, p->q, bp, bm, false);
            }
            // simultaneous (Jacobi) update of every active z
            int64_t upd = 0, deg = 0;
            auto visit = [&](uint64_t z) {
                double nb;
                int r = solve_update(p->bdata[z], bp[z], bm[z], p->Z0, p->beta[z], &nb);
                if (r == 0) { p->beta[z] = p->st(nb); ++upd; }
                else if (r == 2) ++deg;
            };
            if (p->haar3) {
                for (int k = 0; k < (nz >> L); ++k)
                    for (int bi = 0; bi < (ny >> L); ++bi)
                        for (int bj = 0; bj < (nx >> L); ++bj) visit((uint64_t)k * N + (uint64_t)bi * nx + bj);
                for (int l = 1; l <= L; ++l)
                    for (int k = 0; k < (nz >> l); ++k)
                        for (int bi = 0; bi < (ny >> l); ++bi)
                            for (int bj = 0; bj < (nx >> l); ++bj) {
                                if (!active3(p, l, k, bi, bj)) continue;
                                uint64_t z[8];
                                mallat3(nx, ny, nz, l, k, bi, bj, z);
                                for (int t = 1; t < 8; ++t) visit(z[t]);
                            }
            } else {
                for (int s = 0; s < p->nz; ++s) {
                    const uint64_t off = (uint64_t)s * N;
                    for (int bi = 0; bi < (ny >> L); ++bi)
                        for (int bj = 0; bj < (nx >> L); ++bj) visit(off + (uint64_t)bi * nx + bj);
                    for (int l = 1; l <= L; ++l)
                        for (int bi = 0; bi < (ny >> l); ++bi)
                            for (int bj = 0; bj < (nx >> l); ++bj) {
                                if (!is_active(p, l, bi, bj)) continue;
                                BlockIdx z = mallat(nx, ny, l, bi, bj);
                                visit(off + z.H); visit(off + z.V); visit(off + z.D);
                            }
                }
            }
            p->bp_last = bp; p->bm_last = bm;
            p->cum += upd; p->degen += deg;
            std::vector<double> mu = image_of_beta(p, true);
            double obj = refresh_q(p, mu, p->q);
            p->wam_iter++;
            if (recs) {
                recs[it].iter = p->wam_iter;
                recs[it].objective = obj;
                recs[it].elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - p->t0).count();
                recs[it].active_set = p->haar3 ? active_count3(p) : active_count(p);
                recs[it].cum_updates = p->cum;
            }
        }
    })
}

// expand_tree.  2D model: z-summed criterion image
// and a 2D mask shared by all slices.  3D model (pin P3): criterion on every
// voxel, no z-sum; activation of the coarsest inactive 3D block.
int orc_wam_expand(orc_problem* p, double factor, int64_t* newly) {
    ORC_TRY({
        if (!p->wam_ready) throw contract_error("wam: not initialised");
        const int L = p->L, nx = p->g.nx, ny = p->g.ny;
        const uint64_t N = p->Ns;
        std::vector<double> mu = image_of_beta(p, false);   // fp64 criterion image
        std::vector<double> s;
        if (p->haar3) {
            s = mu;
        } else {
            s.assign(N, 0.0);
            for (int sl = 0; sl < p->nz; ++sl)
                for (uint64_t x = 0; x < N; ++x) s[x] += mu[(uint64_t)sl * N + x];
        }
        double mx = -std::numeric_limits<double>::infinity();
        for (double v : s) mx = std::max(mx, v);
        int64_t cnt = 0;
        if (mx > 0.0 && L > 0) {
            const double thr = factor * mx;
            auto na = p->act;
            const int nzs = p->haar3 ? p->g.nz : 1;
            for (int iz = 0; iz < nzs; ++iz)
                for (int iy = 0; iy < ny; ++iy)
                    for (int ix = 0; ix < nx; ++ix) {
                        if (!(s[((uint64_t)iz * ny + iy) * nx + ix] > thr)) continue;
                        for (int l = L; l >= 1; --l) {
                            const std::size_t bidx = p->haar3 ? blk3(p, l, iz >> l, iy >> l, ix >> l)
                                                              : (std::size_t)(iy >> l) * (nx >> l) + (ix >> l);
                            if (!p->act[l][bidx]) {
                                if (!na[l][bidx]) { na[l][bidx] = 1; ++cnt; }
                                break;
                            }
                        }
                    }
            p->act = na;
            if (cnt > 0) {
                compute_z0(p);
                if (p->haar3) build_psi3(p);
                else if (p->mirror) build_nphi(p);
            }
        }
        if (newly) *newly = cnt;
    })
}

int orc_wam_run(orc_problem* p, int iters, const int* sched, int nsched, double factor, orc_record* recs) {
    ORC_TRY({
        for (int it = 1; it <= iters; ++it) {
            int r = orc_wam_iterate(p, 1, recs ? recs + (it - 1) : nullptr);
            if (r != ORC_OK) return r;
            for (int k = 0; k < nsched; ++k)
                if (sched[k] == it) {
                    r = orc_wam_expand(p, factor, nullptr);
                    if (r != ORC_OK) return r;
                    break;
                }
        }
    })
}

int orc_wam_get(const orc_problem* p, double* beta, double* mu, double* q, double* Z0) {
    ORC_TRY({
        if (beta) std::copy(p->beta.begin(), p->beta.end(), beta);
        if (mu) { auto m = image_of_beta(p, true); std::copy(m.begin(), m.end(), mu); }
        if (q) std::copy(p->q.begin(), p->q.end(), q);
        if (Z0) *Z0 = p->Z0;
    })
}

int orc_wam_tree(const orc_problem* p, uint8_t* bits, uint64_t* nbytes) {
    ORC_TRY({
        uint64_t n = 0;
        for (int l = 1; l <= p->L; ++l) {
            if (bits) std::copy(p->act[l].begin(), p->act[l].end(), bits + n);
            n += p->act[l].size();
        }
        if (nbytes) *nbytes = n;
    })
}

int orc_wam_stats(const orc_problem* p, double* b, double* bp, double* bm) {
    ORC_TRY({
        if (b) std::copy(p->bdata.begin(), p->bdata.end(), b);
        if (bp) std::copy(p->bp_last.begin(), p->bp_last.end(), bp);
        if (bm) std::copy(p->bm_last.begin(), p->bm_last.end(), bm);
    })
}

int orc_wam_counters(const orc_problem* p, int64_t* cum, int64_t* degen, int64_t* act) {
    ORC_TRY({
        if (cum) *cum = p->cum;
        if (degen) *degen = p->degen;
        if (act) *act = p->haar3 ? active_count3(p) : active_count(p);
    })
}

int orc_wam_z0_rows(const orc_problem* p, double* zrow) {
    ORC_TRY({
        for (uint64_t y = 0; y < p->Ms; ++y) zrow[y] = p->haar3 ? z_row3(p, y) : z_row(p, y);
    })
}

int orc_phi_column(const orc_problem* p, int L, uint32_t z, uint32_t* rows, double* vals, uint64_t cap,
                   uint64_t* nnz) {
    ORC_TRY({
        const int nx = p->g.nx, ny = p->g.ny;
        check_haar_dims(nx, ny, L);
        uint64_t n = 0;
        for (uint64_t y = 0; y < p->Ms; ++y) {
            double val = 0.0;
            bool hit = false;
            phi_walk(p, L, y, [&](int l, int bi, int bj, double pA, double pH, double pV, double pD) {
                if (L == 0) {
                    if ((uint32_t)(bi * nx + bj) == z) { val = pA; hit = true; }
                    return;
                }
                BlockIdx b = mallat(nx, ny, l, bi, bj);
                if (l == L && b.A == z) { val = pA; hit = true; }
                if (b.H == z) { val = pH; hit = true; }
                if (b.V == z) { val = pV; hit = true; }
                if (b.D == z) { val = pD; hit = true; }
            });
            if (hit && val != 0.0) {
                if (n < cap) { rows[n] = (uint32_t)y; vals[n] = val; }
                ++n;
            }
        }
        *nnz = n;
    })
}

}  // extern "C"
