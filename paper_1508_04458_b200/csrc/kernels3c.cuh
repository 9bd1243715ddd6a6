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

// 2D: mu_c[B] = mu[first pixel of B]; g[x] = G[B(x)] * 4^-k
__global__ void k_mu_coarse2(uint64_t Nc, int nxc, int nx, int k, const float* __restrict__ mu,
                             float* __restrict__ muc) {
    const uint64_t B = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (B >= Nc) return;
    muc[B] = __ldg(mu + ((B / nxc) << k) * (uint64_t)nx + ((B % nxc) << k));
}
__global__ void k_g_expand2(uint64_t N, int nxc, int nx, int k, const double* __restrict__ gc,
                            double* __restrict__ g) {
    const uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= N) return;
    const uint64_t iy = x / nx, ix = x % nx;
    g[x] = __ldg(gc + (iy >> k) * (uint64_t)nxc + (ix >> k)) * (1.0 / (double)(1u << (2 * k)));
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

// ---- z-coarsening on top: the same tree also makes mu constant over groups of
// c = 2^k consecutive slices (the 3D synthesis copies a 2^k-cube's value to all
// its voxels), and the update reads only CUBE sums of g.  So the coarse forward
// runs on nzc = nz / c slices and its line integrals serve every slice of a
// group; the coarse back projection runs on the z-group sums of q, carried as
// two fp32 values (hi = fp32(S), lo = fp32(S - hi): 48 bits of the exact fp64
// sum S of the c fp32 values) because the slab operand is fp32 by design.
__global__ void k_mu_coarse_z(uint64_t Nc, int nxc, int nx, int k, int P, int Pc, int nzc,
                              const float* __restrict__ mu, float* __restrict__ muc) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Nc * (uint64_t)Pc) return;
    const uint64_t B = i / Pc;
    const int zg = (int)(i % Pc);
    const uint64_t x = ((B / nxc) << k) * (uint64_t)nx + ((B % nxc) << k);
    muc[i] = zg < nzc ? __ldg(mu + x * P + ((uint64_t)zg << k)) : 0.f;
}
// debug: mu must equal the value at the first voxel of its 2^k-cube
__global__ void k_mu_coarse_check_z(uint64_t N, int nx, int k, int P, int nz, const float* __restrict__ mu,
                                    int* __restrict__ bad) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N * (uint64_t)nz) return;
    const uint64_t x = i / nz;
    const int s = (int)(i % nz);
    const uint64_t iy = x / nx, ix = x % nx;
    const uint64_t x0 = ((iy >> k) << k) * (uint64_t)nx + ((ix >> k) << k);
    if (__float_as_uint(mu[x * P + s]) != __float_as_uint(mu[x0 * P + ((s >> k) << k)])) atomicOr(bad, 1);
}
// q[y][s] = fp32(I0 exp(-lc[y][s >> k])) and the I-divergence partial of the CTA
// (fixed grid: thread sums in index order, xor butterfly, warps in order)
__global__ void __launch_bounds__(256) k_beer_z(uint64_t M, int nz, int P, int Pc, int k,
                                                const double* __restrict__ lc, const float* __restrict__ I0,
                                                const float* __restrict__ d, float* __restrict__ q,
                                                double* __restrict__ partial, int* __restrict__ flag) {
    double tacc = 0.0;
    const uint64_t n = M * (uint64_t)nz, stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t y = i / nz;
        const int s = (int)(i % nz);
        const double l = lc[y * Pc + (s >> k)];
        if (!isfinite(l)) atomicOr(flag, 1);
        const uint64_t id = y * P + s;
        const double qq = (double)I0[id] * exp(-l);
        q[id] = (float)qq;
        tacc += idiv_term((double)d[id], qq);
    }
    __shared__ double sm[8];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tacc += __shfl_xor_sync(0xffffffffu, tacc, o);
    if (lane == 0) sm[wib] = tacc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += sm[w];
        partial[blockIdx.x] = t;
    }
}
// wz[y][2 zg], wz[y][2 zg + 1] = hi, lo of the slice-order fp64 sum of q over z-group zg
// dbl: the 8 bytes hold the fp64 sum itself (double-operand back projection, k_back3s XD)
__global__ void k_qsum_z(uint64_t M, int nzc, int P, int Pw, int k, int dbl, const float* __restrict__ q,
                         float* __restrict__ wz) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M * (uint64_t)(Pw / 2)) return;
    const uint64_t y = i / (Pw / 2);
    const int zg = (int)(i % (Pw / 2));
    float hi = 0.f, lo = 0.f;
    double S = 0.0;
    if (zg < nzc) {
        const float* p = q + y * P + ((uint64_t)zg << k);
        for (int j = 0; j < (1 << k); ++j) S += (double)__ldg(p + j);
        hi = (float)S;
        lo = (float)(S - (double)hi);
    }
    if (dbl) reinterpret_cast<double*>(wz + y * Pw)[zg] = S;
    else reinterpret_cast<float2*>(wz + y * Pw)[zg] = make_float2(hi, lo);
}
// g[x][s] = (Gc[B][2 zg] + Gc[B][2 zg + 1]) * 8^-k, zg = s >> k: the cube mean on every voxel
// seg > 1: column B was back-projected in seg segments (rows B*seg .. B*seg+seg-1 of gc),
// added here in segment order
__global__ void k_g_expand_z(uint64_t N, int nxc, int nx, int k, int P, int Pw, int nz, int seg,
                             const double* __restrict__ gc, double* __restrict__ g) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N * (uint64_t)nz) return;
    const uint64_t x = i / nz;
    const int s = (int)(i % nz);
    const uint64_t iy = x / nx, ix = x % nx;
    const uint64_t B = (iy >> k) * (uint64_t)nxc + (ix >> k);
    double hi = 0.0, lo = 0.0;
    for (int j = 0; j < seg; ++j) {
        const double2 t = __ldg(reinterpret_cast<const double2*>(gc + (B * seg + j) * Pw) + (s >> k));
        hi += t.x; lo += t.y;
    }
    g[x * P + s] = (hi + lo) * (1.0 / (double)(1u << (3 * k)));
}
// bounds of the column segments: cpseg[B*seg + j] = cp[B] + len_B * j / seg, cpseg[Nc*seg] = cp[Nc]
__global__ void k_seg_bounds(uint64_t Nc, int seg, const unsigned long long* __restrict__ cp,
                             unsigned long long* __restrict__ cpseg) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > Nc * (uint64_t)seg) return;
    if (i == Nc * (uint64_t)seg) { cpseg[i] = cp[Nc]; return; }
    const uint64_t B = i / seg, j = i % seg, lo = cp[B], len = cp[B + 1] - lo;
    cpseg[i] = lo + len * j / seg;
}

}  // namespace wamgpu
