// kernels3c.cuh -- block-coarsened projections of the 3D wavelet-AM iteration.
//
// While the finest active level of the Haar tree is lf > 1, every detail below
// level lf is zero, so mu = Omega beta is constant on the 2^(lf-1) x 2^(lf-1)
// in-plane pixel blocks of every slice (the synthesis applies the same
// operations to every pixel of such a block), and the update reads only
// approximation sums of g = H^T q over those blocks (in WAM
// sum_z phi(y|z) beta(z) = (H idwt(beta))(y)).  With c = 2^(lf-1):
//   l(y, s)  = sum_B Hc(y, B) mu_c(B, s),     Hc(y, B) = sum_{x in B} h(y | x)
//   G(B, s)  = sum_y Hc(y, B) q(y, s)        = sum_{x in B} g(x, s)
// A ray crosses a block in one contiguous run of its Siddon order, so Hc has
// one entry per (ray, block crossed): nnz / ~1.9, ~3.6, ~7 for c = 2, 4, 8.
// Hc values are fp64 ray-order sums of the fp32 h (exact unless a run mixes
// magnitudes more than 2^29 apart), so l and G differ from the pixel path only
// by the association of fp64 sums (~1e-16 relative), like any change of the
// summation order.  The same slab SpMM kernels (k_fwd3s / k_back3s) run over
// the coarse CSR / CSC through the Ent64 entry source.  This is the projector
// used at iterations between expansions lf -> lf - 1; the level-1 phase runs on H.
#pragma once
#include "kernels_phi.cuh"

namespace wamgpu {

__device__ __forceinline__ unsigned coarse_key(unsigned x, int nx, int lgx, bool pow2, int k) {
    int ix, iy;
    if (pow2) { ix = (int)(x & (unsigned)(nx - 1)); iy = (int)(x >> lgx); }
    else { iy = (int)(x / (unsigned)nx); ix = (int)(x % (unsigned)nx); }
    return (unsigned)((iy >> k) * (nx >> k) + (ix >> k));
}

// thread per ray: number of 2^k-blocks it crosses (cnt[M] = 0 for the scan)
__global__ void k_coarse_count(uint64_t M, const unsigned long long* __restrict__ rp, const uint2* __restrict__ A,
                               int nx, int k, unsigned long long* __restrict__ cnt) {
    const uint64_t y = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (y > M) return;
    if (y == M) { cnt[M] = 0; return; }
    const bool pow2 = (nx & (nx - 1)) == 0;
    const int lgx = 31 - __clz(nx);
    unsigned cur = 0xffffffffu;
    unsigned long long c = 0;
    for (uint64_t e = rp[y]; e < rp[y + 1]; ++e) {
        const unsigned key = coarse_key(A[e].x, nx, lgx, pow2, k);
        if (key != cur) { ++c; cur = key; }
    }
    cnt[y] = c;
}

// thread per ray: coarse CSR row (column = block, value = fp64 ray-order sum);
// keys / vals feed the CSC sort (key = block, value = {ray, entry})
__global__ void k_coarse_fill(uint64_t M, const unsigned long long* __restrict__ rp, const uint2* __restrict__ A,
                              int nx, int k, const unsigned long long* __restrict__ rpc, unsigned* __restrict__ colc,
                              double* __restrict__ valc, unsigned* __restrict__ keys, uint2* __restrict__ vals) {
    const uint64_t y = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (y >= M) return;
    const bool pow2 = (nx & (nx - 1)) == 0;
    const int lgx = 31 - __clz(nx);
    uint64_t o = rpc[y];
    unsigned cur = 0xffffffffu;
    double sum = 0.0;
    for (uint64_t e = rp[y]; e < rp[y + 1]; ++e) {
        const uint2 a = A[e];
        const unsigned key = coarse_key(a.x, nx, lgx, pow2, k);
        if (key != cur) {
            if (cur != 0xffffffffu) {
                colc[o] = cur; valc[o] = sum; keys[o] = cur; vals[o] = make_uint2((unsigned)y, (unsigned)o); ++o;
            }
            cur = key;
            sum = 0.0;
        }
        sum = __dadd_rn(sum, hval(a));
    }
    if (cur != 0xffffffffu) {
        colc[o] = cur; valc[o] = sum; keys[o] = cur; vals[o] = make_uint2((unsigned)y, (unsigned)o);
    }
}

// mu_c[B][s] = mu[first pixel of B][s] (mu is constant on B), slab stride P
__global__ void k_mu_coarse(uint64_t Nc, int nxc, int nx, int k, int P, const float* __restrict__ mu,
                            float* __restrict__ muc) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Nc * (uint64_t)(P / 4)) return;
    const uint64_t B = i / (P / 4);
    const int v = (int)(i % (P / 4));
    const uint64_t x = ((B / nxc) << k) * (uint64_t)nx + ((B % nxc) << k);
    reinterpret_cast<float4*>(muc + B * P)[v] = __ldg(reinterpret_cast<const float4*>(mu + x * P) + v);
}

// debug (WAMGPU_COARSE_CHECK=1): flag pixels whose mu differs from their block's first pixel
__global__ void k_mu_coarse_check(uint64_t N, int nx, int k, int P, int nz, const float* __restrict__ mu,
                                  int* __restrict__ bad) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N * (uint64_t)nz) return;
    const uint64_t x = i / nz;
    const int s = (int)(i % nz);
    const uint64_t iy = x / nx, ix = x % nx;
    const uint64_t x0 = ((iy >> k) << k) * (uint64_t)nx + ((ix >> k) << k);
    if (__float_as_uint(mu[x * P + s]) != __float_as_uint(mu[x0 * P + s])) atomicOr(bad, 1);
}

// g[x][s] = G[B(x)][s] * 4^-k: every pixel of B carries the block mean, so the
// Haar analysis of g returns G's approximations exactly (sums of equal values
// and the in-plane 1/2 factors are exact) and zero details below level k + 1
__global__ void k_g_expand(uint64_t N, int nxc, int nx, int k, int P, const double* __restrict__ gc,
                           double* __restrict__ g) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N * (uint64_t)(P / 2)) return;
    const uint64_t x = i / (P / 2);
    const int v = (int)(i % (P / 2));
    const uint64_t iy = x / nx, ix = x % nx;
    const uint64_t B = (iy >> k) * (uint64_t)nxc + (ix >> k);
    const double sc = 1.0 / (double)(1u << (2 * k));
    double2 t = __ldg(reinterpret_cast<const double2*>(gc + B * P) + v);
    t.x *= sc; t.y *= sc;
    reinterpret_cast<double2*>(g + x * P)[v] = t;
}

}  // namespace wamgpu
