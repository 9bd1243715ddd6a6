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

}  // namespace wamgpu
