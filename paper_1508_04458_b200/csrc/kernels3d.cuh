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

// ------------------------------------------------------------ slab SpMM v2
// ncu of slab_dot (profiles/r02_ncu_3d.txt): the XU pipe is 85% busy.  Every
// update converts its fp32 slab value to fp64 with F2F.F64.F32, which runs at
// 4 lanes/clk/SMSP on the XU pipe, and the broadcast h takes one more per
// entry.  v2 removes most of them without changing one bit of the result:
//  * h is converted once per staged entry (per-warp smem), not per lane;
//  * a slab value f is moved into fp64 by integer bit moves, exactly:
//    f2d_scaled(f) = f * 2^-896 for every finite f (normal, zero, denormal:
//    f32 denormals land on fp64 denormals with the same mantissa), and
//    fma(h * 2^896, f2d_scaled(f), acc) == fma(h, (double)f, acc) bit for bit
//    (both products are exactly h*f; FMA rounds once).  NF of every 4 values
//    still take F2F so the XU and ALU pipes share the conversions.
//  * a warp owns G = 32/LPR adjacent rays (voxels), LPR lanes x SPL slices
//    each, stepped in lockstep so neighbouring rays meet the same slab lines
//    close together in time (L1 reuse).
// Summation stays sequential per (ray, slice) in Siddon / CSC order.
template <bool SIGNED>
__device__ __forceinline__ double f2d_scaled(float f) {
    // (One 32x32->64 multiply by 2^29 -- IMAD.WIDE gives both words at once, 1 / 2
    // instructions instead of 2 / 3 -- was measured SLOWER: cfg4 back 1734 vs 1668 ms,
    // forward 2108 vs 2094 ms per run, profiles/r07/ab1.txt; the shifts stay.)
    const unsigned u = __float_as_uint(f);
    const unsigned hi = SIGNED ? (((u & 0x7fffffffu) >> 3) | (u & 0x80000000u)) : (u >> 3);
    return __hiloint2double((int)hi, (int)(u << 29));
}
constexpr double kTwo896 = 0x1p896;

template <int SPL> struct SlabLd {  // SPL consecutive floats as vector loads
    static constexpr int NV = SPL >= 4 ? SPL / 4 : 1;
    using T = typename SlabVec<(SPL >= 4 ? 4 : SPL)>::T;
};
// Lane-to-slice map of the v2 kernels.  SPL <= 2: lane lig owns the SPL
// consecutive slices lig*SPL.. (one load).  SPL >= 4: load i of lane lig is
// the float4 at slice 4*LPR*i + 4*lig, so each load instruction of a group
// covers one contiguous 16*LPR-byte run (full sectors, no sector fetched twice).
template <int LPR, int SPL>
__device__ __forceinline__ int slab_slice(int lig, int j) {
    return SPL >= 4 ? (j / 4) * 4 * LPR + 4 * lig + (j % 4) : lig * SPL + j;
}
template <int LPR, int SPL>
__device__ __forceinline__ void slab_load(const float* p, typename SlabLd<SPL>::T (&v)[SlabLd<SPL>::NV]) {
#pragma unroll
    for (int i = 0; i < SlabLd<SPL>::NV; ++i)
        v[i] = __ldg(reinterpret_cast<const typename SlabLd<SPL>::T*>(p + (SPL >= 4 ? 4 * LPR * i : 0)));
}
template <int SPL>
__device__ __forceinline__ void slab_unpack(const typename SlabLd<SPL>::T (&v)[SlabLd<SPL>::NV], float (&f)[SPL]) {
    if constexpr (SPL >= 4) {
#pragma unroll
        for (int i = 0; i < SPL / 4; ++i) { f[4 * i] = v[i].x; f[4 * i + 1] = v[i].y; f[4 * i + 2] = v[i].z; f[4 * i + 3] = v[i].w; }
    } else {
        float t[SPL];
        unpack(v[0], t);
#pragma unroll
        for (int j = 0; j < SPL; ++j) f[j] = t[j];
    }
}

// per-warp staging: 2 chunk buffers x G groups x K entries (K = 32, 16 for
// G = 8 to stay in 48 KB of static smem per CTA); strides K+4 / K+2 keep the
// G 16-byte broadcasts of a load in distinct bank quads
template <int G> struct SlabStage {
    static constexpr int K = G >= 8 ? 16 : 32, CS = K + 4, HS = K + 2;
    unsigned c[2][G][CS];
    double h[2][G][HS];
};

// acc[j] = sum over entries [lo, hi) of h_k x[idx_k*P + lig*SPL + j]; the
// warp-uniform maxlen is the longest of the warp's G segments (shorter ones
// are padded with h = 0, idx = 0: an exact no-op for finite x).
// Software pipeline: the U gathers of round r+1 are issued before round r is
// consumed (a loop-carried register set, so ptxas cannot sink them), and the
// chunk after the current one is staged into the other smem buffer from
// registers prefetched a whole chunk ahead.
// UX >= 100 selects the ping-pong pipeline (U = UX % 100): two register sets of
// gathered slab values alternate between "in flight" and "being consumed"
// (the round loop is unrolled by two), and h is read from the staged chunk when
// a round is consumed instead of travelling with the gathers.  The copy
// pipeline below moves 40 registers per round (IMAD.MOV: 50 of the 185 SASS
// instructions of a 32-DFMA round at P = 128).
// XD: x is a slab of DOUBLES seen as float pairs (stride P floats = P/2 doubles): the loads
// and the lane-to-slice map are those of the float slab, a lane's SPL floats are SPL/2
// doubles (a float4 chunk = 2 doubles), and acc[0 .. SPL/2) take plain DFMAs with no
// conversion at all (the z-coarse back projection over fp64 z-group sums, kernels3c.cuh).
template <int LPR, int SPL, int UX, int NF, bool SIGNED, int P, bool XD = false, class AP>
__device__ __forceinline__ void slab_dot_g(const AP& A, const float* __restrict__ x, uint64_t lo,
                                           uint64_t hi, int maxlen, int lig, int g,
                                           SlabStage<32 / LPR>& st, double (&acc)[SPL]) {
    constexpr bool PP = UX >= 100;
    constexpr int U = UX % 100;
    constexpr int kSlabK = SlabStage<32 / LPR>::K, NL = kSlabK / LPR, RPC = kSlabK / U;
    static_assert(kSlabK % U == 0 && (U % 4 == 0 || U == 2) && NL >= 1, "unroll");
    using L = SlabLd<SPL>;
#pragma unroll
    for (int j = 0; j < SPL; ++j) acc[j] = 0.0;
    if (maxlen <= 0) return;
    const float* xl = x + slab_slice<LPR, SPL>(lig, 0);
    decltype(ent_zero(A)) nx[NL];
    auto fetch = [&](int base) {
#pragma unroll
        for (int t = 0; t < NL; ++t) {
            const uint64_t k = lo + base + lig + LPR * t;
            nx[t] = k < hi ? ent_ld(A, k) : ent_zero(A);
        }
    };
    auto stage = [&](int buf) {
#pragma unroll
        for (int t = 0; t < NL; ++t) {
            st.c[buf][g][lig + LPR * t] = ent_col(nx[t]);
            st.h[buf][g][lig + LPR * t] = ent_h(nx[t]);
        }
    };
    typename L::T v[U][L::NV];
    double h[U];
    auto issue = [&](int buf, int j0) {   // gathers of the round at entries j0.. of buffer buf
        const unsigned* sc = st.c[buf][g];
        const double* sh = st.h[buf][g];
        if constexpr (U == 2) {
            const uint2 c2 = *reinterpret_cast<const uint2*>(sc + j0);
            const double2 h01 = *reinterpret_cast<const double2*>(sh + j0);
            h[0] = h01.x; h[1] = h01.y;
            slab_load<LPR, SPL>(xl + (uint64_t)c2.x * P, v[0]);
            slab_load<LPR, SPL>(xl + (uint64_t)c2.y * P, v[1]);
        } else {
#pragma unroll
            for (int u = 0; u < U; u += 4) {
                const uint4 c4 = *reinterpret_cast<const uint4*>(sc + j0 + u);
                const double2 h01 = *reinterpret_cast<const double2*>(sh + j0 + u);
                const double2 h23 = *reinterpret_cast<const double2*>(sh + j0 + u + 2);
                h[u] = h01.x; h[u + 1] = h01.y; h[u + 2] = h23.x; h[u + 3] = h23.y;
                slab_load<LPR, SPL>(xl + (uint64_t)c4.x * P, v[u]);
                slab_load<LPR, SPL>(xl + (uint64_t)c4.y * P, v[u + 1]);
                slab_load<LPR, SPL>(xl + (uint64_t)c4.z * P, v[u + 2]);
                slab_load<LPR, SPL>(xl + (uint64_t)c4.w * P, v[u + 3]);
            }
        }
    };
    fetch(0);
    __syncwarp();
    stage(0);
    if (kSlabK < maxlen) fetch(kSlabK);
    __syncwarp();
    const int nr = (maxlen + U - 1) / U;
    if constexpr (PP) {
        static_assert(U % 4 == 0, "ping-pong rounds gather four entries per index load");
        typename L::T va[U][L::NV], vb[U][L::NV];
        auto gather = [&](typename L::T (&vv)[U][L::NV], int r) {   // round r's slab values
            const int chunk = r / RPC, j0 = (r % RPC) * U;
            if (j0 == 0 && r > 0) {   // first round of a new chunk: stage it, prefetch the one after
                stage(chunk & 1);
                if ((chunk + 1) * kSlabK < maxlen) fetch((chunk + 1) * kSlabK);
                __syncwarp();
            }
            const unsigned* sc = st.c[chunk & 1][g];
#pragma unroll
            for (int u = 0; u < U; u += 4) {
                const uint4 c4 = *reinterpret_cast<const uint4*>(sc + j0 + u);
                slab_load<LPR, SPL>(xl + (uint64_t)c4.x * P, vv[u]);
                slab_load<LPR, SPL>(xl + (uint64_t)c4.y * P, vv[u + 1]);
                slab_load<LPR, SPL>(xl + (uint64_t)c4.z * P, vv[u + 2]);
                slab_load<LPR, SPL>(xl + (uint64_t)c4.w * P, vv[u + 3]);
            }
        };
        auto consume = [&](const typename L::T (&vv)[U][L::NV], int r) {
            const int chunk = r / RPC, j0 = (r % RPC) * U;
            const double* sh = st.h[chunk & 1][g] + j0;
#pragma unroll
            for (int u = 0; u < U; u += 2) {
                const double2 h01 = *reinterpret_cast<const double2*>(sh + u);
                const double hp[2] = {h01.x, h01.y};
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    float f[SPL];
                    slab_unpack<SPL>(vv[u + k], f);
                    if constexpr (XD) {
                        static_assert(SPL >= 4 && SPL % 2 == 0, "double operand: float4 chunks");
#pragma unroll
                        for (int j = 0; j < SPL / 2; ++j)
                            acc[j] = fma(hp[k], __hiloint2double(__float_as_int(f[2 * j + 1]), __float_as_int(f[2 * j])),
                                         acc[j]);
                    } else {
                    const double hs = hp[k] * kTwo896;
#pragma unroll
                    for (int j = 0; j < SPL; ++j) {
                        if ((((u + k) * SPL + j) & 3) < NF) acc[j] = fma(hp[k], (double)f[j], acc[j]);
                        else acc[j] = fma(hs, f2d_scaled<SIGNED>(f[j]), acc[j]);
                    }
                    }
                }
            }
        };
        gather(va, 0);
        for (int r = 0; r < nr; r += 2) {
            if (r + 1 < nr) gather(vb, r + 1);
            consume(va, r);
            if (r + 1 < nr) {
                if (r + 2 < nr) gather(va, r + 2);
                consume(vb, r + 1);
            }
        }
        return;
    }
    static_assert(PP || !XD, "double operand: ping-pong pipeline only");
    issue(0, 0);
    // (an explicit two-set ping-pong without these copies was measured slower:
    // 156 registers uncapped, 8.77 vs 8.04 ms at cfg5 with a 128 cap)
    for (int r = 0; r < nr; ++r) {
        typename L::T vc[U][L::NV];
        double hc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            hc[u] = h[u];
#pragma unroll
            for (int i = 0; i < L::NV; ++i) vc[u][i] = v[u][i];
        }
        const int r1 = r + 1;
        if (r1 < nr) {
            const int chunk = r1 / RPC, j0 = (r1 % RPC) * U;
            if (j0 == 0) {   // first round of a new chunk: stage it, prefetch the one after
                stage(chunk & 1);
                if ((chunk + 1) * kSlabK < maxlen) fetch((chunk + 1) * kSlabK);
                __syncwarp();
            }
            issue(chunk & 1, j0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float f[SPL];
            slab_unpack<SPL>(vc[u], f);
            const double hs = hc[u] * kTwo896;
#pragma unroll
            for (int j = 0; j < SPL; ++j) {
                if (((u * SPL + j) & 3) < NF) acc[j] = fma(hc[u], (double)f[j], acc[j]);
                else acc[j] = fma(hs, f2d_scaled<SIGNED>(f[j]), acc[j]);
            }
        }
    }
}

// K2 3D v2: one warp = G adjacent rays (groups of LPR lanes); MODE as k_forward3.
// The warp covers LPR*SPL slices of the stride-P slab per part and loops over
// the parts in [sbeg, nz) (the ray's entries are re-read from L1/L2 per part);
// the host may instead launch once per part (sbeg = part start, nz = its end)
// so that one part's slab columns stay L2-resident (cfg4: 1M voxels x 32 slices
// = 128 MB per part against the 512 MB whole slab).
template <int MODE, int LPR, int SPL, int U, int NF, bool SIGNED, int P, int WPB = 8, int MINB = 1, class AP = const uint2*>
__global__ void __launch_bounds__(32 * WPB, MINB) k_fwd3s(uint64_t M, int sbeg, int nz, const unsigned long long* __restrict__ rp,
                                               AP A, const float* __restrict__ mu,
                                               const float* __restrict__ I0, const float* __restrict__ d,
                                               float* __restrict__ q, double* __restrict__ lout,
                                               double* __restrict__ partial, int* __restrict__ flag) {
    constexpr int G = 32 / LPR, SB = LPR * SPL;
    static_assert(P % SB == 0, "slab parts");
    __shared__ __align__(16) SlabStage<G> s_st[WPB];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, g = lane / LPR, lig = lane % LPR;
    const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    double tacc = 0.0;
    for (uint64_t y0 = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + wib) * G; y0 < M; y0 += W * G)
    for (int s0 = sbeg; s0 < nz; s0 += SB) {
        const uint64_t y = y0 + g;
        const bool ok = y < M;
        const uint64_t lo = ok ? rp[y] : 0, hi = ok ? rp[y + 1] : 0;
        const int maxlen = (int)__reduce_max_sync(0xffffffffu, (unsigned)(hi - lo));
        double acc[SPL];
        slab_dot_g<LPR, SPL, U, NF, SIGNED, P>(A, mu + s0, lo, hi, maxlen, lig, g, s_st[wib], acc);
        if (!ok) continue;
#pragma unroll
        for (int j = 0; j < SPL; ++j) {
            const int s = s0 + slab_slice<LPR, SPL>(lig, j);
            if (s >= nz) continue;
            const uint64_t id = y * P + s;
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

// ---- banded forward (large slabs).  When the slab of mu exceeds L2 (cfg4:
// 1M voxels x 128 slices x 4 B = 512 MB against 126 MB), every view's rays
// sweep the whole image and the gathers go to DRAM (ncu, cfg4 k_fwd3s: 584 GB
// read per launch, 18.7% L2 hits, DRAM 71% busy).  The image is cut into B
// horizontal bands of hb rows (a band's mu is L2-resident); a ray's Siddon
// entries are monotone in iy, so its entries inside band b form one
// contiguous range [blo, bhi) (k_band_bounds).  Band b's launch adds each
// ray's band-b segment to a running fp64 sum per (ray, slice) in lacc, bands
// in fixed order 0..B-1 (deterministic, no atomics); the last band's launch
// finishes as k_fwd3s does (l out, or q = fp32(I0 exp(-l)) + I-div partial).

// per ray y: band b's entries are [rp[y] + blo[y*B + b], rp[y] + bhi[y*B + b])
// (empty bands lo = hi = 0).  Warp per ray; a band boundary is where an
// entry's band differs from its predecessor's.
// bad: set when some row is not monotone in iy (an explicit matrix whose row
// is not in Siddon order): a band would then need several ranges, and the
// caller keeps the unbanded forward.
__global__ void k_band_bounds(uint64_t M, const unsigned long long* __restrict__ rp, const uint2* __restrict__ A,
                              int nx, int hb, int B, unsigned* __restrict__ blo, unsigned* __restrict__ bhi,
                              int* __restrict__ bad) {
    const int lane = threadIdx.x & 31;
    const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t y = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; y < M; y += W) {
        for (int b = lane; b < B; b += 32) { blo[y * B + b] = 0u; bhi[y * B + b] = 0u; }
        __syncwarp();
        const uint64_t lo = rp[y], n = rp[y + 1] - lo;
        for (uint64_t k0 = 0; k0 < n; k0 += 32) {
            const uint64_t k = k0 + lane;
            const int band = k < n ? (int)(A[lo + k].x / (unsigned)nx) / hb : -1;
            const int prev = __shfl_up_sync(0xffffffffu, band, 1);
            int pb = lane ? prev : -1;
            if (lane == 0 && k0) pb = (int)(A[lo + k - 1].x / (unsigned)nx) / hb;
            if (k < n && band != pb) {
                blo[y * B + band] = (unsigned)k;
                if (pb >= 0) bhi[y * B + pb] = (unsigned)k;
            }
            if (k + 1 == n) bhi[y * B + band] = (unsigned)n;
        }
        __syncwarp();
        // every entry in exactly one band range <=> the ranges cover n
        unsigned long long cov = 0;
        for (int b = lane; b < B; b += 32) {
            const unsigned a = blo[y * B + b], e = bhi[y * B + b];
            cov += e >= a ? e - a : (1ull << 40);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) cov += __shfl_xor_sync(0xffffffffu, cov, o);
        if (lane == 0 && cov != n) atomicOr(bad, 1);
        __syncwarp();
    }
}

template <int MODE, int LPR, int SPL, int U, int NF, bool SIGNED, int P, int WPB = 8, int MINB = 1>
__global__ void __launch_bounds__(32 * WPB, MINB) k_fwd3s_band(uint64_t M, int nz, int band, int B,
                                               const unsigned long long* __restrict__ rp,
                                               const unsigned* __restrict__ blo, const unsigned* __restrict__ bhi,
                                               const uint2* __restrict__ A, const float* __restrict__ mu,
                                               const float* __restrict__ I0, const float* __restrict__ d,
                                               float* __restrict__ q, double* __restrict__ lacc,
                                               double* __restrict__ lout, double* __restrict__ partial,
                                               int* __restrict__ flag) {
    constexpr int G = 32 / LPR, SB = LPR * SPL;
    static_assert(P % SB == 0, "slab parts");
    __shared__ __align__(16) SlabStage<G> s_st[WPB];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, g = lane / LPR, lig = lane % LPR;
    const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const bool last = band == B - 1;
    double tacc = 0.0;
    for (uint64_t y0 = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + wib) * G; y0 < M; y0 += W * G)
    for (int s0 = 0; s0 < nz; s0 += SB) {
        const uint64_t y = y0 + g;
        const bool ok = y < M;
        const uint64_t base = ok ? rp[y] : 0;
        const uint64_t lo = ok ? base + blo[y * B + band] : 0, hi = ok ? base + bhi[y * B + band] : 0;
        const int maxlen = (int)__reduce_max_sync(0xffffffffu, (unsigned)(hi - lo));
        if (maxlen == 0 && band > 0 && !last) continue;   // nothing to add anywhere in the warp
        double acc[SPL];
        slab_dot_g<LPR, SPL, U, NF, SIGNED, P>(A, mu + s0, lo, hi, maxlen, lig, g, s_st[wib], acc);
        if (!ok) continue;
#pragma unroll
        for (int j = 0; j < SPL; ++j) {
            const int s = s0 + slab_slice<LPR, SPL>(lig, j);
            if (s >= nz) continue;
            const uint64_t id = y * P + s;
            double tot = acc[j];
            if (band > 0) {
                if (hi == lo && !last) continue;              // nothing to add for this ray
                tot = lacc[id] + acc[j];
            }
            if (!last) {
                lacc[id] = tot;
                continue;
            }
            if (!isfinite(tot)) atomicOr(flag, 1);
            if (MODE == 0) {
                lout[id] = tot;
            } else {
                const double qq = (double)I0[id] * exp(-tot);
                q[id] = (float)qq;
                tacc += idiv_term((double)d[id], qq);
            }
        }
    }
    if (MODE == 1 && last) {
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

// Tile-major layout of the view-group split update (wamgpu.cu tile_update_split):
// the Rv members of a slab own tile rows [r*rows, (r+1)*rows) of the 2^L-cube
// tiles; chunk r of a tile-major buffer holds them, tile (kt, ti, tj) at local
// index ((ti - r*rows)*TX + tj)*TZ + kt, element (i*TS + j)*TS + z.  L = 0: off
// (plain voxel slab / Mallat layout).
struct TileMap {
    int L = 0, TX = 0, TZ = 0, rows = 1, nx = 0, ny = 0, nzl = 0;
    uint64_t CT = 0;   // elements per chunk
};
__device__ __forceinline__ uint64_t tile_elem(const TileMap& m, int iy, int ix, int s) {
    const int TS = 1 << m.L;
    const int ti = iy >> m.L, tj = ix >> m.L, kt = s >> m.L;
    const int r = ti / m.rows;
    const uint64_t lt = ((uint64_t)(ti - r * m.rows) * m.TX + tj) * m.TZ + kt;
    return (uint64_t)r * m.CT + lt * (uint64_t)(TS * TS * TS) +
           (uint64_t)(((iy & (TS - 1)) * TS + (ix & (TS - 1))) * TS + (s & (TS - 1)));
}
// voxel x (= iy*nx + ix), slice s
__device__ __forceinline__ uint64_t tile_pos(const TileMap& m, uint64_t x, int s) {
    return tile_elem(m, (int)(x / (unsigned)m.nx), (int)(x % (unsigned)m.nx), s);
}
// level-l detail coefficient at slab Mallat coordinates (yy, xx, zz): its cube
// position inside the tile holding it (the inverse of kernels3h coef_info3)
__device__ __forceinline__ uint64_t coef_tile_pos(const TileMap& m, int l, int yy, int xx, int zz) {
    const int hl = m.ny >> l, wl = m.nx >> l, dl = m.nzl >> l, sh = m.L - l, half = 1 << sh;
    const int yh = yy >= hl, xh = xx >= wl, zh = zz >= dl;
    const int bi = yy - yh * hl, bj = xx - xh * wl, bk = zz - zh * dl;
    const int i = yh * half + (bi & (half - 1)), j = xh * half + (bj & (half - 1)), z = zh * half + (bk & (half - 1));
    return tile_elem(m, ((bi >> sh) << m.L) + i, ((bj >> sh) << m.L) + j, ((bk >> sh) << m.L) + z);
}

// K3 3D v2: one warp = G voxels of the tile order; MODE as k_back3.
template <int MODE, int LPR, int SPL, int U, int NF, bool SIGNED, int P, int WPB = 8, int MINB = 1, class AP = const uint2*,
          bool XD = false>
__global__ void __launch_bounds__(32 * WPB, MINB) k_back3s(uint64_t N, int sbeg, int nz, const unsigned* __restrict__ order,
                                                const unsigned long long* __restrict__ cp,
                                                AP C, const float* __restrict__ w,
                                                double* __restrict__ g, const double* __restrict__ bam,
                                                float* __restrict__ mu, double Z0, int* __restrict__ flag,
                                                TileMap tmap) {
    constexpr int G = 32 / LPR, SB = LPR * SPL;
    static_assert(P % SB == 0, "slab parts");
    __shared__ __align__(16) SlabStage<G> s_st[WPB];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, gr = lane / LPR, lig = lane % LPR;
    const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i0 = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + wib) * G; i0 < N; i0 += W * G)
    for (int s0 = sbeg; s0 < nz; s0 += SB) {
        const uint64_t i = i0 + gr;
        const bool ok = i < N;
        const uint64_t x = ok ? (order ? order[i] : i) : 0;
        const uint64_t lo = ok ? cp[x] : 0, hi = ok ? cp[x + 1] : 0;
        const int maxlen = (int)__reduce_max_sync(0xffffffffu, (unsigned)(hi - lo));
        double acc[SPL];
        slab_dot_g<LPR, SPL, U, NF, SIGNED, P, XD>(C, w + s0, lo, hi, maxlen, lig, gr, s_st[wib], acc);
        if (!ok) continue;
        if constexpr (XD) {   // MODE 0 only: (sum, 0) in the (hi, lo) slots of the z-group
            static_assert(MODE == 0, "double operand: plain back projection");
#pragma unroll
            for (int j = 0; j < SPL / 2; ++j) {
                const int s = s0 + slab_slice<LPR, SPL>(lig, 2 * j);
                if (s >= nz) continue;
                *reinterpret_cast<double2*>(g + x * P + s) = make_double2(acc[j], 0.0);
            }
            continue;
        }
#pragma unroll
        for (int j = 0; j < SPL; ++j) {
            const int s = s0 + slab_slice<LPR, SPL>(lig, j);
            if (s >= nz) continue;
            const uint64_t id = x * P + s;
            if (MODE == 0) {
                g[tmap.L ? tile_pos(tmap, x, s) : id] = acc[j];   // tile-major: view-group split update
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
// Slab stride P = 32*SPL, or for SPL = 1 any Pr <= 32 (sharded small slabs:
// lanes >= Pr idle).
template <int SPL>
__global__ void __launch_bounds__(256, 4) k_split3(uint64_t nlist, int nz, int Pr, const unsigned* __restrict__ list,
                                                const ulonglong2* __restrict__ col,
                                                const uint2* __restrict__ E, const float* __restrict__ q,
                                                double* __restrict__ bm) {
    using V = typename SlabVec<SPL>::T;
    const int P = SPL == 1 ? Pr : 32 * SPL;
    const int lane = threadIdx.x & 31;
    const bool live = lane * SPL < P;
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
            for (int u = 0; u < U; ++u)
                v[u] = live ? __ldg(reinterpret_cast<const V*>(q + (uint64_t)e[u].x * P) + lane) : V{};
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

// ---- boundary layout transposes on the device (the host only streams
// contiguous rows): reference order [s][i] (n per slice) <-> slab [i][P],
// pad slices zero.  32x32 smem tiles, coalesced on both sides.
template <class T>
__global__ void k_ref_to_slab(const T* __restrict__ src, T* __restrict__ dst, uint64_t n, int nzl, int P) {
    __shared__ T t[32][33];
    const uint64_t i0 = (uint64_t)blockIdx.x * 32;
    const int s0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {   // r: slice within the tile
        const int s = s0 + r;
        const uint64_t i = i0 + threadIdx.x;
        t[r][threadIdx.x] = (s < nzl && i < n) ? src[(uint64_t)s * n + i] : (T)0;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {   // r: element within the tile
        const uint64_t i = i0 + r;
        const int s = s0 + threadIdx.x;
        if (i < n && s < P) dst[i * P + s] = t[threadIdx.x][r];
    }
}
template <class T>
__global__ void k_slab_to_ref(const T* __restrict__ src, T* __restrict__ dst, uint64_t n, int nzl, int P) {
    __shared__ T t[32][33];
    const uint64_t i0 = (uint64_t)blockIdx.x * 32;
    const int s0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const uint64_t i = i0 + r;
        const int s = s0 + threadIdx.x;
        t[threadIdx.x][r] = (i < n && s < nzl) ? src[i * P + s] : (T)0;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int s = s0 + r;
        const uint64_t i = i0 + threadIdx.x;
        if (s < nzl && i < n) dst[(uint64_t)s * n + i] = t[r][threadIdx.x];
    }
}

}  // namespace wamgpu

