// kernels_phi.cuh — projections over the explicit approximation columns Φ_A of
// the 2D Haar tree while no detail coefficient is active (in WAM,
// Σ_z φ(y|z) β(z) ≡ (H·idwt(β))(y)).
//
// With only the level-L approximation roots active, the iteration needs
//   ℓ(y)  = Σ_z φ_A(y|z) β(z)            (instead of H·(Ωβ))
//   S(z)  = Σ_y φ_A(y|z) q̂(y)            (instead of Ωᵀ(Hᵀq̂), approximation z only)
// and b̂₋ = 0 (φ_A ≥ 0).  A ray visits each level-L block in one contiguous run
// of its Siddon order, so Φ_A has one entry per (ray, block crossed): 2.85e7
// entries at cfg2 against 4.5e8 in H.  φ_A follows the quadrant order of the
// expansion walk: q0..q3 are sequential ray-order sums of the
// fp32 h over each quadrant, φ_A = ((q0 + q1) + (q2 + q3)) 2^-L, stored in fp64.
#pragma once
#include "kernels.cuh"

namespace wamgpu {

// Approximation coefficient (Mallat index bi*nx + bj) of cell entry e at level L.
__device__ __forceinline__ unsigned phiA_key(uint2 e, int nx, int lgx, bool pow2, int L) {
    int ix, iy;
    if (pow2) { ix = (int)(e.x & (unsigned)(nx - 1)); iy = (int)(e.x >> lgx); }
    else { iy = (int)(e.x / (unsigned)nx); ix = (int)(e.x % (unsigned)nx); }
    return (unsigned)((iy >> L) * nx + (ix >> L));
}

// thread per ray: number of level-L blocks it crosses (cnt[M] = 0 for the scan)
__global__ void k_phiA_count(uint64_t M, const unsigned long long* __restrict__ rp, const uint2* __restrict__ A,
                             int nx, int L, unsigned long long* __restrict__ cnt) {
    const uint64_t y = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (y > M) return;
    if (y == M) { cnt[M] = 0; return; }
    const bool pow2 = (nx & (nx - 1)) == 0;
    const int lgx = 31 - __clz(nx);
    unsigned cur = 0xffffffffu;
    unsigned long long c = 0;
    for (uint64_t k = rp[y]; k < rp[y + 1]; ++k) {
        const unsigned key = phiA_key(A[k], nx, lgx, pow2, L);
        if (key != cur) { ++c; cur = key; }
    }
    cnt[y] = c;
}

// thread per ray: Φ_A row (CSR) -- column = approximation coefficient, value
// fp64; keys/vals feed the CSC sort (key = column, value = {ray, entry})
__global__ void k_phiA_fill(uint64_t M, const unsigned long long* __restrict__ rp, const uint2* __restrict__ A,
                            int nx, int L, const unsigned long long* __restrict__ rpA, unsigned* __restrict__ colA,
                            double* __restrict__ valA, unsigned* __restrict__ keys, uint2* __restrict__ vals) {
    const uint64_t y = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (y >= M) return;
    const bool pow2 = (nx & (nx - 1)) == 0;
    const int lgx = 31 - __clz(nx);
    const double sc = 1.0 / (double)(1 << L);
    uint64_t o = rpA[y];
    unsigned cur = 0xffffffffu;
    double q[4] = {0.0, 0.0, 0.0, 0.0};
    auto emit = [&]() {
        colA[o] = cur;
        valA[o] = __dmul_rn(__dadd_rn(__dadd_rn(q[0], q[1]), __dadd_rn(q[2], q[3])), sc);
        keys[o] = cur;
        vals[o] = make_uint2((unsigned)y, (unsigned)o);
        ++o;
    };
    for (uint64_t k = rp[y]; k < rp[y + 1]; ++k) {
        const uint2 e = A[k];
        const unsigned key = phiA_key(e, nx, lgx, pow2, L);
        if (key != cur) {
            if (cur != 0xffffffffu) emit();
            cur = key;
            q[0] = q[1] = q[2] = q[3] = 0.0;
        }
        int ix, iy;
        if (pow2) { ix = (int)(e.x & (unsigned)(nx - 1)); iy = (int)(e.x >> lgx); }
        else { iy = (int)(e.x / (unsigned)nx); ix = (int)(e.x % (unsigned)nx); }
        const int quad = (((iy >> (L - 1)) & 1) << 1) | ((ix >> (L - 1)) & 1);
        q[quad] = __dadd_rn(q[quad], hval(e));
    }
    if (cur != 0xffffffffu) emit();
}

// CSC payload after the key sort: rows and values in column order
__global__ void k_phiA_gather(uint64_t n, const uint2* __restrict__ sorted, const double* __restrict__ valA,
                              unsigned* __restrict__ rowC, double* __restrict__ valC) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint2 v = sorted[i];
    rowC[i] = v.x;
    valC[i] = valA[v.y];
}

// S partials: warp per (approximation coefficient a, segment s of SEG) of its
// column; lane-strided fp64 sums, xor butterfly -> part[a*SEG + s]
template <int SEG>
__global__ void __launch_bounds__(256) k_phiA_back(int nA, int wA, int nx, const unsigned long long* __restrict__ cp,
                                                   const unsigned* __restrict__ rowC, const double* __restrict__ valC,
                                                   const float* __restrict__ q, double* __restrict__ part) {
    const int lane = threadIdx.x & 31;
    const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t t = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < (uint64_t)nA * SEG; t += W) {
        const int a = (int)(t / SEG), s = (int)(t % SEG);
        const unsigned z = (unsigned)((a / wA) * nx + (a % wA));
        const uint64_t lo = cp[z], hi = cp[z + 1], len = hi - lo;
        const uint64_t b0 = lo + len * s / SEG, b1 = lo + len * (s + 1) / SEG;
        double acc = 0.0;
        for (uint64_t k = b0 + lane; k < b1; k += 32) acc = fma(valC[k], (double)__ldg(q + rowC[k]), acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) part[t] = acc;
    }
}

// approximation update (k_tile mode 1 restricted to the active roots): S from
// the SEG partials in fixed order, b- = 0, the same solve_update and counters
template <int SEG>
__global__ void k_phiA_update(int nA, int wA, int nx, const double* __restrict__ part,
                              const double* __restrict__ bdata, float* __restrict__ beta, double Z0,
                              double* __restrict__ bp_out, double* __restrict__ bm_out,
                              unsigned long long* __restrict__ counters, int* __restrict__ flag) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long upd = 0, deg = 0;
    if (a < nA) {
        const unsigned z = (unsigned)((a / wA) * nx + (a % wA));
        double S = 0.0;
        for (int s = 0; s < SEG; ++s) S += part[(uint64_t)a * SEG + s];
        if (bp_out) { bp_out[z] = S; bm_out[z] = 0.0; }
        double nb;
        const int rr = solve_update(bdata[z], S, 0.0, Z0, (double)beta[z], &nb);
        if (rr == 0) {
            if (!isfinite(nb)) atomicOr(flag, 4);
            beta[z] = (float)nb;
            upd = 1;
        } else if (rr == 2) {
            deg = 1;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        upd += __shfl_xor_sync(0xffffffffu, upd, o);
        deg += __shfl_xor_sync(0xffffffffu, deg, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (upd) atomicAdd(counters + 0, upd);
        if (deg) atomicAdd(counters + 1, deg);
    }
}

// ℓ = Φ_A β fused with q = fp32(I0 e^-ℓ) and the I-divergence partial
// (k_fwd_patch's epilogue); 8 lanes per ray, 4 rays per warp
__global__ void __launch_bounds__(256) k_phiA_fwd(uint64_t M, const unsigned long long* __restrict__ rpA,
                                                  const unsigned* __restrict__ colA, const double* __restrict__ valA,
                                                  const float* __restrict__ beta, const float* __restrict__ I0,
                                                  const float* __restrict__ d, float* __restrict__ q,
                                                  double* __restrict__ partial, int* __restrict__ flag) {
    constexpr int LPR = 8, R = 4;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, sub = lane % LPR;
    const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t ntask = (M + R - 1) / R;
    double tacc = 0.0;
    for (uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + wib; t < ntask; t += W) {
        const uint64_t y = t * R + lane / LPR;
        const bool has = y < M;
        uint64_t lo = 0, hi = 0;
        if (has) { lo = rpA[y]; hi = rpA[y + 1]; }
        double acc = 0.0;
        for (uint64_t k = lo + sub; k < hi; k += LPR) acc = fma(valA[k], (double)__ldg(beta + colA[k]), acc);
#pragma unroll
        for (int o = LPR / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (has && sub == 0) {
            if (!isfinite(acc)) atomicOr(flag, 1);
            const double qq = (double)I0[y] * exp(-acc);
            q[y] = (float)qq;
            tacc += idiv_term((double)d[y], qq);
        }
    }
    __shared__ double s[32];
    double v = tacc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) s[wib] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tt = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tt += s[w];
        partial[blockIdx.x] = tt;
    }
}

// ---- separable 3D Haar (pin P3) on the axial stack ----------------------------
// The approximation column of in-plane block b and z-block k factorises
// (kernels3h.cuh): φ(y_s | b,k) = φ_A(y|b) c^L for the slices s of z-block k
// (s >> L == k), 0 elsewhere; φ_A is the 2D in-plane column above.  So the
// in-plane Φ_A serves every slice:
//   ℓ(y,s) = c^L Σ_b φ_A(y|b) β(b, s >> L)
//   S(b,k) = c^L Σ_y φ_A(y|b) Σ_{s >> L == k} q̂(y,s)
// Slabs are [ray or voxel][P] (slice fastest); lane j of a warp owns slices
// j*SPL .. j*SPL + SPL - 1.
// The forward multiplies the raw block sums of h (φ_A 2^L, exact) by mblk(b,k)
// = fp32(Ωβ) on the block, the value the synthesis writes into μ for a lone
// approximation coefficient: per level v <- (v c) 0.5, the operation order of
// cube_inv.  So ℓ equals the H path's Σ h μ up to the fp64 summation order
// (a fp64 c^L product would differ from the fp32 μ by ~1e-7).

// ℓ = Σ_b (φ_A 2^L) mblk(b, s >> L) over one ray per warp, fused with q̂ and
// the I-divergence partial
template <int SPL>
__global__ void __launch_bounds__(256) k_phiA3_fwd(uint64_t M, int nzl, int P, int L, int nx, int wA,
                                                   const unsigned long long* __restrict__ rpA,
                                                   const unsigned* __restrict__ colA, const double* __restrict__ valA,
                                                   const float* __restrict__ mblk, const float* __restrict__ I0,
                                                   const float* __restrict__ d, float* __restrict__ q,
                                                   double* __restrict__ partial, int* __restrict__ flag) {
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const int NK = nzl >> L;
    const double s2L = (double)(1 << L);
    double tacc = 0.0;
    for (uint64_t y = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; y < M; y += W) {
        const uint64_t lo = rpA[y], hi = rpA[y + 1];
        double acc[SPL];
#pragma unroll
        for (int j = 0; j < SPL; ++j) acc[j] = 0.0;
        for (uint64_t b0 = lo; b0 < hi; b0 += 32) {
            const int n = (int)(hi - b0 < 32 ? hi - b0 : 32);
            unsigned al = 0;
            double vl = 0.0;
            if (lane < n) {
                const unsigned col = colA[b0 + lane];
                al = (col / (unsigned)nx) * (unsigned)wA + (col % (unsigned)nx);
                vl = valA[b0 + lane] * s2L;   // raw block sum of h (exact)
            }
            for (int i = 0; i < n; ++i) {
                const unsigned a = __shfl_sync(0xffffffffu, al, i);
                const double v = __shfl_sync(0xffffffffu, vl, i);
                const float* mp = mblk + (uint64_t)a * NK;
#pragma unroll
                for (int j = 0; j < SPL; ++j) {
                    const int s = lane * SPL + j;
                    if (s < nzl) acc[j] = fma(v, (double)__ldg(mp + (s >> L)), acc[j]);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < SPL; ++j) {
            const int s = lane * SPL + j;
            if (s >= nzl) continue;
            const double lg = acc[j];
            if (!isfinite(lg)) atomicOr(flag, 1);
            const uint64_t id = y * P + s;
            const double qq = (double)I0[id] * exp(-lg);
            q[id] = (float)qq;
            tacc += idiv_term((double)d[id], qq);
        }
    }
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

// fp32(Ωβ) of a lone approximation coefficient (cube_inv's operation order)
__device__ __forceinline__ float synth_root3(float beta, int L) {
    double v = (double)beta;
    for (int l = L; l >= 1; --l) v = __dmul_rn(__dmul_rn(v, 0.70710678118654752440), 0.5);
    return (float)v;
}

// S partials: warp per (in-plane block a, segment s) of its column; each lane
// sums its slices, the lanes of a z-block combine by an xor butterfly
// (2^L / SPL lanes per z-block) -> part[(a*SEG + s)*NK + k], NK = nzl >> L
template <int SEG, int SPL>
__global__ void __launch_bounds__(256) k_phiA3_back(int nA, int wA, int nx, int nzl, int P, int L,
                                                    const unsigned long long* __restrict__ cp,
                                                    const unsigned* __restrict__ rowC, const double* __restrict__ valC,
                                                    const float* __restrict__ q, double* __restrict__ part) {
    const int lane = threadIdx.x & 31;
    const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const int NK = nzl >> L;
    const int lpk = max(1, (1 << L) / SPL);   // lanes per z-block
    for (uint64_t t = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < (uint64_t)nA * SEG; t += W) {
        const int a = (int)(t / SEG), sg = (int)(t % SEG);
        const unsigned z = (unsigned)((a / wA) * nx + (a % wA));
        const uint64_t lo = cp[z], hi = cp[z + 1], len = hi - lo;
        const uint64_t b0 = lo + len * sg / SEG, b1 = lo + len * (sg + 1) / SEG;
        double acc = 0.0;   // this lane's slices summed (all in one z-block: SPL <= 2^L)
        for (uint64_t k = b0; k < b1; ++k) {
            const double v = valC[k];
            const float* qp = q + (uint64_t)rowC[k] * P;
            double sq = 0.0;
#pragma unroll
            for (int j = 0; j < SPL; ++j) {
                const int s = lane * SPL + j;
                if (s < nzl) sq += (double)__ldg(qp + s);
            }
            acc = fma(v, sq, acc);
        }
        for (int o = 1; o < lpk; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const int s0 = lane * SPL;
        if (s0 < nzl && (lane % lpk) == 0) part[((uint64_t)a * SEG + sg) * NK + (s0 >> L)] = acc;
    }
}

// approximation update of the separable 3D model: S(b,k) = c^L x the fixed-order
// sum of the segment partials; b- = 0; the same solve_update and counters
template <int SEG>
__global__ void k_phiA3_update(int nA, int wA, int nx, int NK, int P, int L, double cL,
                               const double* __restrict__ part, const double* __restrict__ bdata,
                               float* __restrict__ beta, float* __restrict__ mblk, double Z0,
                               double* __restrict__ bp_out, double* __restrict__ bm_out,
                               unsigned long long* __restrict__ counters, int* __restrict__ flag) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long upd = 0, deg = 0;
    if (e < (uint64_t)nA * NK) {
        const int a = (int)(e / NK), k = (int)(e % NK);
        const uint64_t z = ((uint64_t)(a / wA) * nx + (a % wA)) * P + k;
        double S = 0.0;
        for (int s = 0; s < SEG; ++s) S += part[((uint64_t)a * SEG + s) * NK + k];
        S *= cL;
        if (bp_out) { bp_out[z] = S; bm_out[z] = 0.0; }
        double nb;
        const int rr = solve_update(bdata[z], S, 0.0, Z0, (double)beta[z], &nb);
        if (rr == 0) {
            if (!isfinite(nb)) atomicOr(flag, 4);
            beta[z] = (float)nb;
            upd = 1;
        } else if (rr == 2) {
            deg = 1;
        }
        mblk[e] = synth_root3(beta[z], L);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        upd += __shfl_xor_sync(0xffffffffu, upd, o);
        deg += __shfl_xor_sync(0xffffffffu, deg, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (upd) atomicAdd(counters + 0, upd);
        if (deg) atomicAdd(counters + 1, deg);
    }
}

}  // namespace wamgpu
