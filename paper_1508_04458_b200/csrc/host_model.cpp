// host_model.cpp — host-side parts of libwamgpu.so (product code, not the oracle).
//
//  * ray table for the device Siddon tracer: the reference's make_ray arithmetic
//    (proj/include/wamrec/projector.hpp:22-49; uniform_angles geometry.hpp:70-74)
//    evaluated with host libm so the rays are bit-identical to the reference's;
//    plus the pinned equiangular arc detector (P1).  Built with
//    -ffp-contract=off (an FMA changes the rays).
//  * phantom-sim: painter's-order rasterisation with voxel-centre
//    inclusion and seeded Poisson data from a counter-based generator
//    (splitmix64 keyed by (seed, ray, draw); inversion below mean 12, PTRS
//    transformed rejection above).  Runs once per problem on the host in f64
//    with exact ray/voxel lengths traced on the fly (projector.hpp:64-119).
#include "host_model.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numbers>
#include <stdexcept>
#include <thread>
#include <vector>

namespace wamgpu {

std::vector<double> view_angles(const wamgpu_geometry& g) {
    std::vector<double> a((std::size_t)g.views);
    if (g.view_angles) {
        for (int v = 0; v < g.views; ++v) a[v] = g.view_angles[v];
    } else {
        const double arc = g.beam == WAMGPU_BEAM_PARALLEL ? std::numbers::pi : 2.0 * std::numbers::pi;
        for (int v = 0; v < g.views; ++v) a[v] = arc * v / g.views;
    }
    return a;
}

void validate(const wamgpu_geometry& g) {  // geometry.hpp:51-67
    if (g.nx < 4 || g.ny < 4) throw ConfigError("geometry: nx and ny must be >= 4");
    if (g.nz < 1) throw ConfigError("geometry: nz must be >= 1");
    if (!(g.voxel_size > 0.0)) throw ConfigError("geometry: voxel_size must be positive");
    if (g.detectors < 1) throw ConfigError("geometry: at least one detector required");
    if (g.views < 1) throw ConfigError("geometry: at least one view required");
    if (g.beam < 0 || g.beam > 2) throw ConfigError("geometry: unknown beam type");
    if (g.beam != WAMGPU_BEAM_FAN_ARC && !(g.detector_spacing > 0.0))
        throw ConfigError("geometry: detector_spacing must be positive");
    if (g.view_angles)
        for (int v = 0; v < g.views; ++v)
            if (!std::isfinite(g.view_angles[v])) throw ConfigError("geometry: non-finite view angle");
    if (g.beam != WAMGPU_BEAM_PARALLEL) {
        if (!(g.source_to_center > 0.0)) throw ConfigError("geometry: source_to_center must be positive");
        if (!(g.source_to_detector > g.source_to_center))
            throw ConfigError("geometry: source_to_detector must exceed source_to_center");
    }
    if (g.beam == WAMGPU_BEAM_FAN_ARC && !(g.fan_angle_step > 0.0))
        throw ConfigError("geometry: fan_angle_step must be positive");
}

std::vector<RayD> ray_table(const wamgpu_geometry& g) {
    validate(g);
    const std::vector<double> ang = view_angles(g);
    const int V = g.views, D = g.detectors;
    std::vector<RayD> rays((std::size_t)V * D);
    for (int v = 0; v < V; ++v) {
        const double theta = ang[v];
        const double c = std::cos(theta), s = std::sin(theta);
        for (int k = 0; k < D; ++k) {
            RayD r{};
            if (g.beam == WAMGPU_BEAM_PARALLEL) {
                const double u = (k - 0.5 * (D - 1)) * g.detector_spacing;
                r.ox = -s * u; r.oy = c * u; r.dx = c; r.dy = s;
                r.tmin = -std::numeric_limits<double>::max();
                r.tmax = std::numeric_limits<double>::max();
            } else if (g.beam == WAMGPU_BEAM_FAN_FLAT) {
                const double u = (k - 0.5 * (D - 1)) * g.detector_spacing;
                const double sx = g.source_to_center * c, sy = g.source_to_center * s;
                const double px = sx - g.source_to_detector * c - s * u;
                const double py = sy - g.source_to_detector * s + c * u;
                const double len = std::hypot(px - sx, py - sy);
                r.ox = sx; r.oy = sy; r.dx = (px - sx) / len; r.dy = (py - sy) / len;
                r.tmin = 0.0; r.tmax = len;
            } else {
                const double gam = (k - 0.5 * (D - 1)) * g.fan_angle_step;
                const double cg = std::cos(gam), sg = std::sin(gam);
                r.ox = g.source_to_center * c; r.oy = g.source_to_center * s;
                r.dx = -c * cg - s * sg;
                r.dy = -s * cg + c * sg;
                r.tmin = 0.0; r.tmax = g.source_to_detector;
            }
            rays[(std::size_t)v * D + k] = r;
        }
    }
    return rays;
}

// Siddon traversal, projector.hpp:52-119 (host copy used only by the simulator;
// the iteration's matrix comes from the device tracer in kernels.cuh).
template <typename Emit>
static void trace_host(int nx, int ny, double h, const RayD& ray, Emit&& emit) {
    const double W = nx * h, Hh = ny * h;
    const double xmin = -0.5 * W, ymin = -0.5 * Hh;
    double tmin = ray.tmin, tmax = ray.tmax;
    auto clip = [&](double o, double d, double lo, double hi) {
        if (d == 0.0) return o >= lo && o <= hi;
        double t0 = (lo - o) / d, t1 = (hi - o) / d;
        if (t0 > t1) std::swap(t0, t1);
        if (t0 > tmin) tmin = t0;
        if (t1 < tmax) tmax = t1;
        return tmin < tmax;
    };
    if (!clip(ray.ox, ray.dx, xmin, xmin + W)) return;
    if (!clip(ray.oy, ray.dy, ymin, ymin + Hh)) return;
    if (!(tmax > tmin)) return;
    auto cell = [](double pos, double origin, double edge, int n) {
        int i = static_cast<int>(std::floor((pos - origin) / edge));
        return std::clamp(i, 0, n - 1);
    };
    const double ex = ray.ox + tmin * ray.dx, ey = ray.oy + tmin * ray.dy;
    int ix = cell(ex, xmin, h, nx), iy = cell(ey, ymin, h, ny);
    const int sx = ray.dx > 0.0 ? 1 : -1, sy = ray.dy > 0.0 ? 1 : -1;
    const double big = std::numeric_limits<double>::max();
    const double dtx = ray.dx != 0.0 ? h / std::abs(ray.dx) : big;
    const double dty = ray.dy != 0.0 ? h / std::abs(ray.dy) : big;
    double nxt = big, nyt = big;
    if (ray.dx != 0.0) { double e = xmin + (ray.dx > 0.0 ? ix + 1 : ix) * h; nxt = (e - ray.ox) / ray.dx; }
    if (ray.dy != 0.0) { double e = ymin + (ray.dy > 0.0 ? iy + 1 : iy) * h; nyt = (e - ray.oy) / ray.dy; }
    double t = tmin;
    while (t < tmax) {
        double ts = std::min({nxt, nyt, tmax});
        double len = ts - t;
        if (len > 0.0) emit(ix, iy, len);
        if (ts >= tmax) break;
        if (nxt <= ts) { ix += sx; nxt += dtx; if (ix < 0 || ix >= nx) break; }
        if (nyt <= ts) { iy += sy; nyt += dty; if (iy < 0 || iy >= ny) break; }
        t = ts;
    }
}

static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static inline double uniform01(uint64_t seed, uint64_t stream, uint64_t k) {
    uint64_t x = mix64(mix64(seed) ^ mix64(stream * 0x100000001B3ull + k));
    return ((double)(x >> 11) + 0.5) * 0x1.0p-53;
}
static double poisson(uint64_t seed, uint64_t stream, double m) {
    if (!(m >= 0.0) || !std::isfinite(m)) throw NumericError("simulate: invalid Poisson mean");
    if (m == 0.0) return 0.0;
    if (m < 12.0) {
        double u = uniform01(seed, stream, 0);
        double p = std::exp(-m), F = p, k = 0.0;
        while (u > F && k < 1000.0) { k += 1.0; p *= m / k; F += p; }
        return k;
    }
    const double slam = std::sqrt(m), loglam = std::log(m);
    const double b = 0.931 + 2.53 * slam, a = -0.059 + 0.02483 * b;
    const double invalpha = 1.1239 + 1.1328 / (b - 3.4), vr = 0.9277 - 3.6224 / (b - 2.0);
    for (uint64_t j = 0;; ++j) {
        double U = uniform01(seed, stream, 2 * j + 1) - 0.5;
        double V = uniform01(seed, stream, 2 * j + 2);
        double us = 0.5 - std::fabs(U);
        double k = std::floor((2.0 * a / us + b) * U + m + 0.43);
        if (us >= 0.07 && V <= vr) return k;
        if (k < 0.0 || (us < 0.013 && V > us)) continue;
        if (std::log(V) + std::log(invalpha) - std::log(a / (us * us) + b) <= -m + k * loglam - std::lgamma(k + 1.0))
            return k;
    }
}

void rasterize(const wamgpu_geometry& g, const wamgpu_primitive* pr, int np, double bg, double* mu) {
    validate(g);
    const double h = g.voxel_size;
    const double x0 = -0.5 * (g.nx * h), y0 = -0.5 * (g.ny * h), z0 = -0.5 * (g.nz * h);
    for (int iz = 0; iz < g.nz; ++iz)
        for (int iy = 0; iy < g.ny; ++iy)
            for (int ix = 0; ix < g.nx; ++ix) {
                const double x = x0 + (ix + 0.5) * h, y = y0 + (iy + 0.5) * h, z = z0 + (iz + 0.5) * h;
                double v = bg;
                for (int i = 0; i < np; ++i) {
                    const wamgpu_primitive& q = pr[i];
                    if (q.value < 0.0) throw ConfigError("phantom: attenuation must be >= 0");
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
}

void simulate(const wamgpu_geometry& g, const double* mu, const double* I0, uint64_t seed, bool noisy, int threads,
              double* d) {
    const std::vector<RayD> rays = ray_table(g);
    const uint64_t M = rays.size(), N = (uint64_t)g.nx * g.ny;
    int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
    nt = (int)std::min<uint64_t>((uint64_t)nt, M);
    std::vector<std::thread> pool;
    std::vector<std::string> errs(nt);
    const uint64_t chunk = (M + nt - 1) / nt;
    for (int b = 0; b < nt; ++b) {
        pool.emplace_back([&, b] {
            try {
                const uint64_t lo = b * chunk, hi = std::min(M, lo + chunk);
                std::vector<std::pair<uint32_t, double>> row;
                for (uint64_t y = lo; y < hi; ++y) {
                    row.clear();
                    trace_host(g.nx, g.ny, g.voxel_size, rays[y], [&](int ix, int iy, double len) {
                        row.push_back({(uint32_t)iy * (uint32_t)g.nx + (uint32_t)ix, len});
                    });
                    for (int s = 0; s < g.nz; ++s) {
                        double acc = 0.0;
                        for (auto& e : row) acc += e.second * mu[(uint64_t)s * N + e.first];
                        const uint64_t id = (uint64_t)s * M + y;
                        const double m = I0[id] * std::exp(-acc);
                        d[id] = noisy ? poisson(seed, id, m) : m;
                    }
                }
            } catch (const std::exception& e) { errs[b] = e.what(); }
        });
    }
    for (auto& t : pool) t.join();
    for (auto& e : errs)
        if (!e.empty()) throw NumericError(e);
}

}  // namespace wamgpu
