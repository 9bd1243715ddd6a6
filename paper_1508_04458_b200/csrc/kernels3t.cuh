// kernels3t.cuh — the on-the-fly 3D forward projector of the north_star:
// l[y][s] = sum_x h(y|x) mu[x][s] for an axial stack (pin P2), with h computed
// on the fly by the device Siddon tracer (projector.hpp:52-119, the same
// fp64 operations as trace_dev / the stored matrix, so fp32(h) and the
// ray-order fp64 sums are bit-identical to the stored-H slab SpMM k_fwd3s) and
// the image tile staged in shared memory by TMA (cp.async.bulk.tensor).
//
// Why tiles: the slab SpMM gathers every (entry, slice) value from L1/L2 and
// moves 2.4 B per ray-voxel update from L2 (ncu, cfg4: 579 GB per launch =
// 9.4 TB/s, ~80% of the ~6300 B/clk L2 cap): it is L2-bandwidth-bound.  Here a
// CTA owns a BUNDLE of 512/CB adjacent views x CB adjacent channels (512
// rays that cross the same image strip) for one chunk of 32 slices and marches
// along the bundle's major axis in steps of T3_TW pixels.  For every step one
// elected thread issues the TMA loads of the [minor rows x T3_TW columns x 32
// slices] box the bundle crosses (a 3D tensor map over mu[y][x][s], zero fill
// outside the image), double-buffered against an mbarrier pair, so each mu
// value is fetched from L2 once per bundle step and then read 4-11 times from
// shared memory.
//
// Per step every thread advances the Siddon state of ITS ray through the
// step's columns and writes (tile pixel, fp32 h) into a per-ray ring; then the
// warp consumes its 32 rays four at a time (8 lanes x 4 slices per ray:
// conflict-free 128-byte LDS per ray) with sequential fp64 FMAs per (ray,
// slice) in Siddon order.  Accumulators stay in registers over the whole march.
#pragma once
#include <cuda.h>
#include "kernels3d.cuh"

namespace wamgpu {

constexpr int T3_RAYS = 512;  // rays (threads) per bundle: CB adjacent channels x 512/CB adjacent views
constexpr int T3_TW = 4;      // major-axis pixels per step
constexpr int T3_ZB = 32;     // slices per CTA
constexpr int T3_RB = 32;     // minor-axis pixels per TMA box
constexpr int T3_NBOX = 5;    // boxes per step buffer (minor extent <= 160)
constexpr int T3_CAP = 12;    // ring entries per ray per step
constexpr int T3_BOXPIX = T3_TW * T3_RB;
constexpr int T3_BUFPIX = T3_BOXPIX * T3_NBOX;
constexpr int T3_WARPS = T3_RAYS / 32;

struct T3Smem {
    float buf[2][T3_BUFPIX][T3_ZB];          // 2 x 80 KB, TMA destinations
    uint2 ring[T3_CAP][T3_RAYS];             // per ray per step: x = byte offset of the tile pixel | low 3 h bits << 29,
                                             //                   y = high word of double(h * 2^896)
    int cnt[T3_RAYS];
    double oray[32][4];                      // outer rays (ox, oy, dx, dy) of every view (<= 16 views)
    unsigned long long full[2], empty[2];    // mbarriers
    int hdr[2][4];                           // per buffer: minor origin, major origin, boxes
    int kmin, kmax, nalive;
    double red[T3_WARPS];
};

// error bits raised in flag (the host then keeps the stored-H slab SpMM):
//   0x100 box taller than T3_NBOX*T3_RB   0x200 ray against the bundle's march direction
//   0x400 entry outside the staged box    0x800 ray alive after the march / barrier timeout
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_wait(unsigned long long* b, unsigned parity) {
    const unsigned a = smem_u32(b);
    for (unsigned i = 0; i < (1u << 22); ++i) {
        unsigned ok;
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(a), "r"(parity) : "memory");
        if (ok) return true;
    }
    return false;   // bounded: a lost TMA must not hang the GPU
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2,
                                            unsigned long long* bar) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(smem_u32(dst)), "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)) : "memory");
}

// Resumable Siddon state of one ray: init() is trace_dev's prologue, next()
// one turn of its loop (same operations in the same order, explicit _rn).
struct T3Trace {
    double t, tmax, nxt, nyt, dtx, dty;
    int ix, iy, sx, sy;
    bool alive;
    __device__ __forceinline__ void init(int nx, int ny, double h, const RayDev& r, int& ixe, int& iye) {
        alive = false;
        ixe = iye = 0;
        const double W = __dmul_rn((double)nx, h), Hh = __dmul_rn((double)ny, h);
        const double xmin = __dmul_rn(-0.5, W), ymin = __dmul_rn(-0.5, Hh);
        double tmin = r.tmin;
        tmax = r.tmax;
        if (!clip_axis_dev(r.ox, r.dx, xmin, __dadd_rn(xmin, W), tmin, tmax)) return;
        if (!clip_axis_dev(r.oy, r.dy, ymin, __dadd_rn(ymin, Hh), tmin, tmax)) return;
        if (!(tmax > tmin)) return;
        const double ex = __dadd_rn(r.ox, __dmul_rn(tmin, r.dx));
        const double ey = __dadd_rn(r.oy, __dmul_rn(tmin, r.dy));
        ix = (int)floor(__ddiv_rn(__dsub_rn(ex, xmin), h));
        iy = (int)floor(__ddiv_rn(__dsub_rn(ey, ymin), h));
        ix = min(max(ix, 0), nx - 1);
        iy = min(max(iy, 0), ny - 1);
        sx = r.dx > 0.0 ? 1 : -1;
        sy = r.dy > 0.0 ? 1 : -1;
        const double big = DBL_MAX;
        dtx = r.dx != 0.0 ? __ddiv_rn(h, fabs(r.dx)) : big;
        dty = r.dy != 0.0 ? __ddiv_rn(h, fabs(r.dy)) : big;
        nxt = big; nyt = big;
        if (r.dx != 0.0) {
            double e = __dadd_rn(xmin, __dmul_rn((double)(r.dx > 0.0 ? ix + 1 : ix), h));
            nxt = __ddiv_rn(__dsub_rn(e, r.ox), r.dx);
        }
        if (r.dy != 0.0) {
            double e = __dadd_rn(ymin, __dmul_rn((double)(r.dy > 0.0 ? iy + 1 : iy), h));
            nyt = __ddiv_rn(__dsub_rn(e, r.oy), r.dy);
        }
        t = tmin;
        alive = t < tmax;
        // exit cell estimate (march bound only; the trace itself decides)
        const double fx = __dadd_rn(r.ox, __dmul_rn(tmax, r.dx)), fy = __dadd_rn(r.oy, __dmul_rn(tmax, r.dy));
        ixe = min(max((int)floor(__ddiv_rn(__dsub_rn(fx, xmin), h)), 0), nx - 1);
        iye = min(max((int)floor(__ddiv_rn(__dsub_rn(fy, ymin), h)), 0), ny - 1);
    }
    // one turn: returns the length in the current cell (<= 0: nothing to emit)
    // and moves to the next cell; call only while alive
    __device__ __forceinline__ double next(int nx, int ny, int& cx, int& cy) {
        const double ts = fmin(fmin(nxt, nyt), tmax);
        const double len = __dsub_rn(ts, t);
        cx = ix; cy = iy;
        if (ts >= tmax) { alive = false; return len; }
        if (nxt <= ts) { ix += sx; nxt = __dadd_rn(nxt, dtx); if (ix < 0 || ix >= nx) alive = false; }
        if (alive && nyt <= ts) { iy += sy; nyt = __dadd_rn(nyt, dty); if (iy < 0 || iy >= ny) alive = false; }
        t = ts;
        return len;
    }
};

struct T3Args {
    const RayDev* rays;      // local rays, row y = v*D + ch
    int V, D;                // local views, channels per view
    int nx, ny, nzl, P;
    double h;
    const float* I0; const float* d;
    float* q; double* lout; double* partial; int* flag;
};

// MODE 0: l (fp64) out; MODE 1: q = fp32(I0 exp(-l)) + I-divergence partial per CTA.
// NF of every 4 slab values are converted by F2F, the rest by the exact bit
// move (kernels3d.cuh f2d_scaled); h never takes a conversion: the tracer
// stores the words of double(h * 2^896) (h = fp32(len) is a positive normal
// float: high word (bits >> 3) + (1792 << 20), low word bits << 29).
// CB channels x VG = 512/CB views per bundle.
template <int MODE, int NF, bool SIGNED, int CB>
__global__ void __launch_bounds__(T3_RAYS, 1) k_fwd3t(const __grid_constant__ CUtensorMap tmx,
                                                      const __grid_constant__ CUtensorMap tmy, T3Args a) {
    constexpr int VG = T3_RAYS / CB;
    static_assert(VG >= 1 && 2 * VG <= 32, "bundle shape");
    extern __shared__ __align__(128) unsigned char t3_raw[];
    T3Smem& S = *reinterpret_cast<T3Smem*>(t3_raw);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int ncb = (a.D + CB - 1) / CB, nvg = (a.V + VG - 1) / VG;
    const int cbn = blockIdx.x % ncb, vg = (blockIdx.x / ncb) % nvg, zc = blockIdx.x / (ncb * nvg);
    const int s0 = zc * T3_ZB, v0 = vg * VG, c0 = cbn * CB;
    const int vi = tid / CB, ci = tid % CB;
    const bool valid = v0 + vi < a.V && c0 + ci < a.D;
    const uint64_t y = (uint64_t)(v0 + vi) * a.D + (c0 + ci);

    // bundle major axis and direction from its central ray
    const RayDev rc = a.rays[(uint64_t)min(v0 + VG / 2, a.V - 1) * a.D + min(c0 + CB / 2, a.D - 1)];
    const bool xmaj = fabs(rc.dx) >= fabs(rc.dy);
    const int smaj = (xmaj ? rc.dx : rc.dy) > 0.0 ? 1 : -1;
    const int nmaj = xmaj ? a.nx : a.ny, nmin = xmaj ? a.ny : a.nx;
    const double W = __dmul_rn((double)a.nx, a.h), Hh = __dmul_rn((double)a.ny, a.h);
    const double xmin = __dmul_rn(-0.5, W), ymin = __dmul_rn(-0.5, Hh);

    if (tid == 0) {
        S.kmin = 1 << 30; S.kmax = -1; S.nalive = 0;
        mbar_init(&S.full[0], 1); mbar_init(&S.full[1], 1);
        mbar_init(&S.empty[0], T3_WARPS); mbar_init(&S.empty[1], T3_WARPS);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (tid < 2 * VG) {   // outer rays of every view of the bundle
        const int vv = min(v0 + (tid >> 1), a.V - 1), cc = (tid & 1) ? min(c0 + CB - 1, a.D - 1) : c0;
        const RayDev r = a.rays[(uint64_t)vv * a.D + cc];
        S.oray[tid][0] = r.ox; S.oray[tid][1] = r.oy; S.oray[tid][2] = r.dx; S.oray[tid][3] = r.dy;
    }
    __syncthreads();

    T3Trace tr;
    tr.alive = false;
    if (valid) {
        const RayDev r = a.rays[y];
        int ixe, iye;
        tr.init(a.nx, a.ny, a.h, r, ixe, iye);
        if (tr.alive) {
            const int sm = xmaj ? tr.sx : tr.sy;
            if (sm != smaj) { atomicOr(a.flag, 0x200); tr.alive = false; }
        }
        if (tr.alive) {
            const int c_in = xmaj ? tr.ix : tr.iy, c_out = xmaj ? ixe : iye;
            const int m_in = smaj > 0 ? c_in : nmaj - 1 - c_in, m_out = smaj > 0 ? c_out : nmaj - 1 - c_out;
            atomicMin(&S.kmin, m_in / T3_TW);
            atomicMax(&S.kmax, min(max(m_out, m_in) + 1, nmaj - 1) / T3_TW);
            atomicAdd(&S.nalive, 1);
        }
    }
    __syncthreads();
    const int kmin = S.kmin, kmax = S.kmax;
    double acc[8][4];
#pragma unroll
    for (int g = 0; g < 8; ++g)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[g][j] = 0.0;

    // producer (warp 0): box of step k into buffer b.  Lane l < 2 VG holds an
    // outer ray (first / last channel of view l >> 1) and evaluates it at the
    // two planes bounding the step; the box is the min/max over them +- 1.
    auto produce = [&](int k, int b) {
        const int ma = smaj > 0 ? k * T3_TW : nmaj - (k + 1) * T3_TW;   // lowest real major index of the step
        int lo = 1 << 30, hi = -(1 << 30);
        if (lane < 2 * VG) {
            const double ox = S.oray[lane][0], oy = S.oray[lane][1], dx = S.oray[lane][2], dy = S.oray[lane][3];
#pragma unroll
            for (int pl = 0; pl < 2; ++pl) {
                const double e = (xmaj ? xmin : ymin) + (double)(ma + pl * T3_TW) * a.h;
                const double tp = xmaj ? (e - ox) / dx : (e - oy) / dy;
                const double mv = xmaj ? oy + tp * dy : ox + tp * dx;
                const double f = floor((mv - (xmaj ? ymin : xmin)) / a.h);
                const int r = (int)fmin(fmax(f, -1.0e6), 1.0e6);
                lo = min(lo, r); hi = max(hi, r);
            }
        }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        lo = max(lo - 1, 0); hi = min(hi + 1, nmin - 1);
        int nb = hi >= lo ? (hi - lo) / T3_RB + 1 : 0;
        if (nb > T3_NBOX) { if (lane == 0) atomicOr(a.flag, 0x100); nb = T3_NBOX; }
        if (lane == 0) {
            S.hdr[b][0] = lo; S.hdr[b][1] = ma; S.hdr[b][2] = nb;
            if (nb == 0) {
                mbar_arrive(&S.full[b]);
            } else {
                mbar_expect_tx(&S.full[b], (unsigned)nb * T3_BOXPIX * T3_ZB * 4u);
                for (int j = 0; j < nb; ++j) {
                    if (xmaj) tma_load_3d(&S.buf[b][j * T3_BOXPIX][0], &tmx, s0, ma, lo + j * T3_RB, &S.full[b]);
                    else tma_load_3d(&S.buf[b][j * T3_BOXPIX][0], &tmy, s0, lo + j * T3_RB, ma, &S.full[b]);
                }
            }
        }
        __syncwarp();
    };

    if (S.nalive > 0) {
        if (w == 0) {
            produce(kmin, 0);
            if (kmin + 1 <= kmax) produce(kmin + 1, 1);
        }
        const int sub = lane >> 3, lig = lane & 7;
        for (int k = kmin; k <= kmax; ++k) {
            const int b = (k - kmin) & 1;
            const unsigned ph = (unsigned)((k - kmin) >> 1) & 1u;
            if (!mbar_wait(&S.full[b], ph)) atomicOr(a.flag, 0x800);
            const int lo = S.hdr[b][0], ma = S.hdr[b][1], nb = S.hdr[b][2];
            // ---- trace this ray through the step's columns, at most T3_CAP
            // cells per round (steep rays of wide bundles take several rounds),
            // then consume the warp's 32 rings
            const unsigned char* bb = reinterpret_cast<const unsigned char*>(&S.buf[b][0][0]) + lig * 16;
            const int mend = (k + 1) * T3_TW;
            bool more;
            do {
                int n = 0;
                bool pend = false;
                while (tr.alive) {
                    const int cm = xmaj ? tr.ix : tr.iy;
                    const int m = smaj > 0 ? cm : nmaj - 1 - cm;
                    if (m >= mend) break;
                    if (n >= T3_CAP) { pend = true; break; }
                    int cx, cy;
                    const double len = tr.next(a.nx, a.ny, cx, cy);
                    if (len > 0.0) {
                        const int mi = (xmaj ? cy : cx) - lo, mj = (xmaj ? cx : cy) - ma;
                        unsigned pix;
                        if (xmaj) pix = (unsigned)(mi * T3_TW + mj);
                        else pix = (unsigned)((mi >> 5) * T3_BOXPIX + mj * T3_RB + (mi & 31));
                        const unsigned hb = __float_as_uint((float)len);
                        if (mi < 0 || mi >= nb * T3_RB || mj < 0 || mj >= T3_TW || (hb >> 23) == 0u) {
                            if (hb) atomicOr(a.flag, 0x400);   // outside the box, or a denormal h (h = 0 adds nothing)
                            continue;
                        }
                        S.ring[n][tid] = make_uint2((pix * (unsigned)(T3_ZB * 4)) | (hb << 29), (hb >> 3) + 0x70000000u);
                        ++n;
                    }
                }
                S.cnt[tid] = n;
                more = __any_sync(0xffffffffu, pend);
                __syncwarp();
                // 8 groups of 4 rays, 8 lanes x 4 slices per ray; the ring entry two
                // turns ahead and the slab values one turn ahead are in flight
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    const int rl = w * 32 + g * 4 + sub;
                    const int ne = S.cnt[rl];
                    uint2 e0 = S.ring[0][rl], e1 = S.ring[1][rl];
                    float4 mc = *reinterpret_cast<const float4*>(bb + (e0.x & 0x1ff80u));
                    for (int e = 0; e < ne; ++e) {
                        const float4 mn = *reinterpret_cast<const float4*>(bb + (e1.x & 0x1ff80u));
                        const uint2 e2 = S.ring[min(e + 2, T3_CAP - 1)][rl];
                        const int lw = (int)(e0.x & 0xe0000000u);
                        const double hs = __hiloint2double((int)e0.y, lw);
                        const double hh = __hiloint2double((int)(e0.y - 0x38000000u), lw);
                        const float f[4] = {mc.x, mc.y, mc.z, mc.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            if (j < NF) acc[g][j] = fma(hh, (double)f[j], acc[g][j]);
                            else acc[g][j] = fma(hs, f2d_scaled<SIGNED>(f[j]), acc[g][j]);
                        }
                        e0 = e1; e1 = e2; mc = mn;
                    }
                }
                __syncwarp();
            } while (more);
            if (lane == 0) mbar_arrive(&S.empty[b]);
            if (w == 0 && k + 2 <= kmax) {
                if (!mbar_wait(&S.empty[b], ph)) atomicOr(a.flag, 0x800);
                produce(k + 2, b);
            }
        }
        if (tr.alive) atomicOr(a.flag, 0x800);
    }

    // ---- outputs: lane (sub, lig) holds ray w*32 + g*4 + sub, slices s0 + lig*4 + j
    double tacc = 0.0;
    {
        const int sub = lane >> 3, lig = lane & 7;
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const int rl = w * 32 + g * 4 + sub;
            const int rv = v0 + rl / CB, rch = c0 + rl % CB;
            if (rv >= a.V || rch >= a.D) continue;
            const uint64_t yy = (uint64_t)rv * a.D + rch;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int s = s0 + lig * 4 + j;
                if (s >= a.nzl) continue;
                const uint64_t id = yy * a.P + s;
                if (!isfinite(acc[g][j])) atomicOr(a.flag, 1);
                if (MODE == 0) {
                    a.lout[id] = acc[g][j];
                } else {
                    const double qq = (double)a.I0[id] * exp(-acc[g][j]);
                    a.q[id] = (float)qq;
                    tacc += idiv_term((double)a.d[id], qq);
                }
            }
        }
    }
    if (MODE == 1) {
        double v = tacc;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) S.red[w] = v;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int i = 0; i < T3_WARPS; ++i) t += S.red[i];
            a.partial[blockIdx.x] = t;
        }
    }
}

}  // namespace wamgpu
