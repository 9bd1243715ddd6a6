// kernels3d.cuh — the axial 3D stack (nz > 1 slices sharing one in-plane
// system matrix, geometry.hpp:17-20; pin P2).
//
// Every ray y of the in-plane matrix is traced once and reused for all nz
// slices, so each projector pass is a sparse-matrix x dense-slab product:
// one WARP per in-plane ray (forward) or voxel (back), the matrix entry is a
// warp-uniform (broadcast) load and the lanes cover the slices of a z-fastest
// slab (SPL slices per lane: nz <= P = 32 SPL), so every gather is one
// coalesced P*4-byte segment.  Device layouts (stride P): mu3/beta3 [x][s]
// fp32, q3/d3/I03 [y][s] fp32, g3/bdata3/bm3 [z][s] fp64.  The boundary transposes to the reference
// layouts (image.hpp:14 (z*ny+iy)*nx+ix, rays z*M+y).
#pragma once
#include "kernels.cuh"

namespace wamgpu {

// Slab stride P = 32*SPL (device layouts are padded to it; pad slices are
// zero and carry I0 = d = 0, so they contribute nothing): every lane owns SPL
// consecutive slices and all slab loads are unconditional vector loads.
template <int SPL> struct SlabVec;
template <> struct SlabVec<1> { using T = float; };
template <> struct SlabVec<2> { using T = float2; };
template <> struct SlabVec<4> { using T = float4; };
__device__ __forceinline__ void unpack(float v, float (&o)[1]) { o[0] = v; }
__device__ __forceinline__ void unpack(float2 v, float (&o)[2]) { o[0] = v.x; o[1] = v.y; }
__device__ __forceinline__ void unpack(float4 v, float (&o)[4]) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }

// Slab SpMV of one row/column: acc[j] = sum_k h_k x[idx_k*P + lane*SPL + j].
// The warp loads 32 matrix entries with ONE coalesced load (lane j holds entry
// base+j), prefetches the next 32 while it works, broadcasts entries by
// shuffle, and keeps 8 slab gathers in flight per lane.
template <int SPL>
__device__ __forceinline__ void slab_dot(const uint2* __restrict__ A, const float* __restrict__ x, uint64_t lo,
                                         uint64_t hi, int lane, double (&acc)[SPL]) {
    using V = typename SlabVec<SPL>::T;
    constexpr int P = 32 * SPL;
#pragma unroll
    for (int j = 0; j < SPL; ++j) acc[j] = 0.0;
    uint2 cur = (lo + lane < hi) ? ld_stream(A + lo + lane) : make_uint2(0u, 0u);
    for (uint64_t base = lo; base < hi; base += 32) {
        const uint64_t nb = base + 32;
        const uint2 nxt = (nb + lane < hi) ? ld_stream(A + nb + lane) : make_uint2(0u, 0u);
        const int n = (int)((hi - base) < 32 ? (hi - base) : 32);
        for (int j0 = 0; j0 < n; j0 += 8) {
            unsigned c[8];
            float h[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                c[u] = __shfl_sync(0xffffffffu, cur.x, j0 + u);
                h[u] = __uint_as_float(__shfl_sync(0xffffffffu, cur.y, j0 + u));
            }
            V v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(reinterpret_cast<const V*>(x + (uint64_t)c[u] * P) + lane);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                float f[SPL];
                unpack(v[u], f);
                const double hh = (double)h[u];
#pragma unroll
                for (int j = 0; j < SPL; ++j) acc[j] = fma(hh, (double)f[j], acc[j]);
            }
        }
        cur = nxt;
    }
}

// K2 3D: l[y][s] = sum_x h(y|x) mu[x][s]; MODE 0 writes l (fp64, [y][s]);
// MODE 1 fuses q = fp32(I0 exp(-l)) and the fp64 I-divergence partial.
template <int MODE, int SPL>
__global__ void __launch_bounds__(256, 4) k_forward3(uint64_t M, int nz, const unsigned long long* __restrict__ rp,
                                                  const uint2* __restrict__ A, const float* __restrict__ mu,
                                                  const float* __restrict__ I0, const float* __restrict__ d,
                                                  float* __restrict__ q, double* __restrict__ lout,
                                                  double* __restrict__ partial, int* __restrict__ flag) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    double tacc = 0.0;
    for (uint64_t y = (uint64_t)blockIdx.x * (blockDim.x >> 5) + wib; y < M; y += W) {
        double acc[SPL];
        slab_dot<SPL>(A, mu, rp[y], rp[y + 1], lane, acc);
#pragma unroll
        for (int j = 0; j < SPL; ++j) {
            const int s = lane * SPL + j;
            if (s >= nz) continue;
            const uint64_t id = y * (32 * SPL) + s;
            if (!isfinite(acc[j])) atomicOr(flag, 1);
            if (MODE == 0) {
                lout[id] = acc[j];
            } else {
                const double qq = (double)I0[id] * exp(-acc[j]);
                q[id] = (float)qq;
                tacc += idiv_term((double)d[id], qq);
            }
        }
    }
    if (MODE == 1) {
        __shared__ double sm[32];
        double v = tacc;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) sm[wib] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sm[w];
            partial[blockIdx.x] = t;
        }
    }
}

// K3 3D: g[x][s] = sum_y h(y|x) w[y][s] over the voxel's CSC column (no
// atomics).  MODE 0: g (fp64).  MODE 1: fused AM update of mu[x][s]
// (SPEC.md:303, 316-317).  Voxels are visited in 2D tile order (`order`) so the
// concurrently processed columns share rays and the q-slab gathers hit L2.
template <int MODE, int SPL>
__global__ void __launch_bounds__(256, 4) k_back3(uint64_t N, int nz, const unsigned* __restrict__ order,
                                               const unsigned long long* __restrict__ cp, const uint2* __restrict__ C,
                                               const float* __restrict__ w, double* __restrict__ g,
                                               const double* __restrict__ bam, float* __restrict__ mu, double Z0,
                                               int* __restrict__ flag) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = (uint64_t)blockIdx.x * (blockDim.x >> 5) + wib; i < N; i += W) {
        const uint64_t x = order ? order[i] : i;
        double acc[SPL];
        slab_dot<SPL>(C, w, cp[x], cp[x + 1], lane, acc);
#pragma unroll
        for (int j = 0; j < SPL; ++j) {
            const int s = lane * SPL + j;
            if (s >= nz) continue;
            const uint64_t id = x * (32 * SPL) + s;
            if (MODE == 0) {
                g[id] = acc[j];
            } else {
                const double b = bam[id], c = acc[j];
                if (b > 0.0 && c > 0.0) {
                    const double v = (double)mu[id] + log(c / b) / Z0;
                    if (!isfinite(v)) atomicOr(flag, 2);
                    mu[id] = (float)((0.0 < v) ? v : 0.0);
                }
            }
        }
    }
}

// K5 3D: b-[z][s] = sum over the (slice-shared) Phi^- column of z of q[y][s] phi,
// exact 2^-20 fixed-point accumulation per slice (order-independent, as k_split).
template <int SPL>
__global__ void __launch_bounds__(256, 4) k_split3(uint64_t nlist, int nz, const unsigned* __restrict__ list,
                                                const ulonglong2* __restrict__ col,
                                                const uint2* __restrict__ E, const float* __restrict__ q,
                                                double* __restrict__ bm) {
    using V = typename SlabVec<SPL>::T;
    constexpr int P = 32 * SPL;
    const int lane = threadIdx.x & 31;
    const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nlist; i += W) {
        const unsigned z = list[i];
        const ulonglong2 cr = col[z];
        const uint64_t lo = cr.x, hi = cr.y;
        long long acc[SPL];
#pragma unroll
        for (int j = 0; j < SPL; ++j) acc[j] = 0;
        constexpr int U = 8;
        for (uint64_t k0 = lo; k0 < hi; k0 += U) {
            uint2 e[U];
#pragma unroll
            for (int u = 0; u < U; ++u) e[u] = __ldg(E + (k0 + u < hi ? k0 + u : lo));
            V v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = __ldg(reinterpret_cast<const V*>(q + (uint64_t)e[u].x * P) + lane);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (k0 + u >= hi) break;
                float f[SPL];
                unpack(v[u], f);
                const double ph = hval(e[u]);
#pragma unroll
                for (int j = 0; j < SPL; ++j) acc[j] += fix_term((double)f[j], ph);
            }
        }
#pragma unroll
        for (int j = 0; j < SPL; ++j) {
            const int s = lane * SPL + j;
            if (s < nz) bm[(uint64_t)z * P + s] = (double)acc[j] * kFixInv;
        }
    }
}

// Haar tiles of a slab: one CTA per (2^L x 2^L tile, chunk of sc slices); every
// level step works on all sc slices at once (one __syncthreads per step, not
// per slice).  Same per-2x2 operation order as k_tile.
// mode 0: synthesis beta -> mu (and mu64); mode 1: analysis + root solve +
// synthesis; mode 2: analysis only (g -> out).  Slab stride P.
__device__ __forceinline__ void tiles_fwd(double* x, double* t, int TS, int L, int ns) {
    const int T2 = TS * TS;
    for (int l = 1; l <= L; ++l) {
        const int s = TS >> (l - 1), h2 = s >> 1, g2 = h2 * h2;
        for (int i = threadIdx.x; i < g2 * ns; i += blockDim.x) {
            const int sl = i / g2, r = i % g2, gi = r / h2, gj = r % h2;
            const double* xs = x + sl * T2;
            double* ts = t + sl * T2;
            const double a = xs[(2 * gi) * TS + 2 * gj], b = xs[(2 * gi) * TS + 2 * gj + 1];
            const double c = xs[(2 * gi + 1) * TS + 2 * gj], d = xs[(2 * gi + 1) * TS + 2 * gj + 1];
            const double s1 = a + b, s2 = c + d, d1 = a - b, d2 = c - d;
            ts[gi * TS + gj] = (s1 + s2) * 0.5;
            ts[(gi + h2) * TS + gj] = (s1 - s2) * 0.5;
            ts[gi * TS + gj + h2] = (d1 + d2) * 0.5;
            ts[(gi + h2) * TS + gj + h2] = (d1 - d2) * 0.5;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < s * s * ns; i += blockDim.x) {
            const int sl = i / (s * s), r = i % (s * s);
            x[sl * T2 + (r / s) * TS + r % s] = t[sl * T2 + (r / s) * TS + r % s];
        }
        __syncthreads();
    }
}
__device__ __forceinline__ void tiles_inv(double* x, double* t, int TS, int L, int ns) {
    const int T2 = TS * TS;
    for (int l = L; l >= 1; --l) {
        const int s = TS >> (l - 1), h2 = s >> 1, g2 = h2 * h2;
        for (int i = threadIdx.x; i < g2 * ns; i += blockDim.x) {
            const int sl = i / g2, r = i % g2, gi = r / h2, gj = r % h2;
            const double* xs = x + sl * T2;
            double* ts = t + sl * T2;
            const double A = xs[gi * TS + gj], H = xs[(gi + h2) * TS + gj];
            const double V = xs[gi * TS + gj + h2], D = xs[(gi + h2) * TS + gj + h2];
            const double p = A + H, m = A - H, r2 = V + D, u = V - D;
            ts[(2 * gi) * TS + 2 * gj] = (p + r2) * 0.5;
            ts[(2 * gi) * TS + 2 * gj + 1] = (p - r2) * 0.5;
            ts[(2 * gi + 1) * TS + 2 * gj] = (m + u) * 0.5;
            ts[(2 * gi + 1) * TS + 2 * gj + 1] = (m - u) * 0.5;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < s * s * ns; i += blockDim.x) {
            const int sl = i / (s * s), r = i % (s * s);
            x[sl * T2 + (r / s) * TS + r % s] = t[sl * T2 + (r / s) * TS + r % s];
        }
        __syncthreads();
    }
}

__global__ void k_tile3(int mode, int nx, int ny, int nz, int P, int L, int sc, const double* __restrict__ g,
                        const double* __restrict__ bm, const double* __restrict__ bdata,
                        const uint8_t* __restrict__ act, ActOff off, float* __restrict__ beta,
                        float* __restrict__ mu, double* __restrict__ mu64, double* __restrict__ out,
                        double* __restrict__ bp_out, double* __restrict__ bm_out, double Z0,
                        unsigned long long* __restrict__ counters, int* __restrict__ flag) {
    extern __shared__ double sm3[];
    const int TS = 1 << L, T2 = TS * TS;
    const int ti = blockIdx.y, tj = blockIdx.x, s0 = blockIdx.z * sc;
    const int ns = min(sc, nz - s0);
    double* xs = sm3;                 // [sc][T2]
    double* ts = sm3 + sc * T2;       // [sc][T2] scratch
    const uint64_t base = (uint64_t)ti * TS * nx + (uint64_t)tj * TS;
    // voxel-major, slices fastest: contiguous ns*8-byte runs per voxel
    if (mode != 0) {
        for (int i = threadIdx.x; i < T2 * ns; i += blockDim.x) {
            const int v = i / ns, s = i % ns;
            xs[s * T2 + v] = g[(base + (uint64_t)(v / TS) * nx + v % TS) * P + s0 + s];
        }
        __syncthreads();
        tiles_fwd(xs, ts, TS, L, ns);
    }
    if (mode == 2) {
        for (int i = threadIdx.x; i < T2 * ns; i += blockDim.x) {
            const int v = i / ns, s = i % ns;
            CoefInfo ci = coef_info(v / TS, v % TS, ti, tj, L, nx, ny, act, off);
            out[ci.z * P + s0 + s] = xs[s * T2 + v];
        }
        return;
    }
    unsigned long long upd = 0, deg = 0;
    for (int i = threadIdx.x; i < T2 * ns; i += blockDim.x) {
        const int v = i / ns, s = i % ns;
        CoefInfo ci = coef_info(v / TS, v % TS, ti, tj, L, nx, ny, act, off);
        const uint64_t zid = ci.z * P + s0 + s;
        float bo = beta[zid];
        if (mode == 1) {
            const double bmv = ci.approx ? 0.0 : bm[zid];
            const double bpv = xs[s * T2 + v] - bmv;
            if (bp_out) { bp_out[zid] = bpv; bm_out[zid] = bmv; }
            if (ci.active) {
                double nb;
                const int r = solve_update(bdata[zid], bpv, bmv, Z0, (double)bo, &nb);
                if (r == 0) {
                    if (!isfinite(nb)) atomicOr(flag, 4);
                    bo = (float)nb;
                    beta[zid] = bo;
                    ++upd;
                } else if (r == 2) {
                    ++deg;
                }
            }
        }
        xs[s * T2 + v] = (double)bo;
    }
    if (mode == 1) {
        for (int o = 16; o > 0; o >>= 1) {
            upd += __shfl_xor_sync(0xffffffffu, upd, o);
            deg += __shfl_xor_sync(0xffffffffu, deg, o);
        }
        if ((threadIdx.x & 31) == 0) {
            if (upd) atomicAdd(counters + 0, upd);
            if (deg) atomicAdd(counters + 1, deg);
        }
    }
    __syncthreads();
    tiles_inv(xs, ts, TS, L, ns);
    for (int i = threadIdx.x; i < T2 * ns; i += blockDim.x) {
        const int v = i / ns, s = i % ns;
        const uint64_t p = (base + (uint64_t)(v / TS) * nx + v % TS) * P + s0 + s;
        mu[p] = (float)xs[s * T2 + v];
        if (mu64) mu64[p] = xs[s * T2 + v];
    }
}

// z-summed criterion image: s(p) = sum_s mu64[p][s] in slice order.
__global__ void k_zsum(uint64_t N, int nz, int P, const double* __restrict__ mu64, double* __restrict__ out) {
    const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= N) return;
    double s = 0.0;
    for (int k = 0; k < nz; ++k) s += mu64[p * P + k];
    out[p] = s;
}

}  // namespace wamgpu
