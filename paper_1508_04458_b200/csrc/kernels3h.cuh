// kernels3h.cuh — separable 3D Haar model of the wavelet AM (pin P3,
// SURVEY.md App. A) on the axial 3D stack: octree of 2^l x 2^l x 2^l blocks, 7
// details per node, criterion on every voxel (no z-sum).
//
// A level-l coefficient's column factorises (rays never leave their slice):
//   phi(y_s | z) = psi_p(y | b) * c^l * sigma(s)
// with psi_p (p in A,H,V,D) the in-plane quadrant combination of the 2D model
// (DESIGN.md §4), c = 1/sqrt(2) and sigma = +1 (z low-pass) or +-1 on the two
// z-halves of the block (z high-pass).  So the expansion walk stays in-plane,
// one Psi entry (ray, psi_A, psi_H, psi_V, psi_D) per (ray, in-plane block b)
// serves every z-block of b, and the split needs slab sums of q over z-halves.
// Coefficients use the slab-local 3D Mallat layout stored as [yy*nx+xx][zz]
// (stride P), like images.
#pragma once
#include "kernels3d.cuh"

namespace wamgpu {

constexpr double kC3 = 0.70710678118654752440;
__device__ __forceinline__ double cpow3(int l) {  // c^l by repeated multiplication (oracle: cpow3)
    double c = 1.0;
    for (int i = 0; i < l; ++i) c *= kC3;
    return c;
}

// ------------------------------------------------------------ 3D Haar tiles
// smem cube x[z][i][j] (TS^3).  One level on the leading s^3 region: per
// 2x2x2 group the in-plane step on both z-planes (DESIGN.md §3 order), then
// low = (P0+P1)*c, high = (P0-P1)*c at planes k and k + s/2.
__device__ __forceinline__ void cube_fwd(double* x, double* t, int TS, int L) {
    for (int l = 1; l <= L; ++l) {
        const int s = TS >> (l - 1), h2 = s >> 1, g3 = h2 * h2 * h2;
        for (int i = threadIdx.x; i < g3; i += blockDim.x) {
            const int k = i / (h2 * h2), r = i % (h2 * h2), gi = r / h2, gj = r % h2;
            double P[2][4];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const double* xp = x + (2 * k + e) * TS * TS;
                const double a = xp[(2 * gi) * TS + 2 * gj], b = xp[(2 * gi) * TS + 2 * gj + 1];
                const double c = xp[(2 * gi + 1) * TS + 2 * gj], d = xp[(2 * gi + 1) * TS + 2 * gj + 1];
                const double s1 = a + b, s2 = c + d, d1 = a - b, d2 = c - d;
                P[e][0] = (s1 + s2) * 0.5; P[e][1] = (s1 - s2) * 0.5;
                P[e][2] = (d1 + d2) * 0.5; P[e][3] = (d1 - d2) * 0.5;
            }
            const int pi[4] = {gi, gi + h2, gi, gi + h2}, pj[4] = {gj, gj, gj + h2, gj + h2};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                t[(k * TS + pi[q]) * TS + pj[q]] = (P[0][q] + P[1][q]) * kC3;
                t[((k + h2) * TS + pi[q]) * TS + pj[q]] = (P[0][q] - P[1][q]) * kC3;
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < s * s * s; i += blockDim.x) {
            const int z = i / (s * s), r = i % (s * s), ii = r / s, jj = r % s;
            x[(z * TS + ii) * TS + jj] = t[(z * TS + ii) * TS + jj];
        }
        __syncthreads();
    }
}
__device__ __forceinline__ void cube_inv(double* x, double* t, int TS, int L) {
    for (int l = L; l >= 1; --l) {
        const int s = TS >> (l - 1), h2 = s >> 1, g3 = h2 * h2 * h2;
        for (int i = threadIdx.x; i < g3; i += blockDim.x) {
            const int k = i / (h2 * h2), r = i % (h2 * h2), gi = r / h2, gj = r % h2;
            const int pi[4] = {gi, gi + h2, gi, gi + h2}, pj[4] = {gj, gj, gj + h2, gj + h2};
            double P[2][4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double lo = x[(k * TS + pi[q]) * TS + pj[q]], hi = x[((k + h2) * TS + pi[q]) * TS + pj[q]];
                P[0][q] = (lo + hi) * kC3;
                P[1][q] = (lo - hi) * kC3;
            }
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                double* tp = t + (2 * k + e) * TS * TS;
                const double A = P[e][0], H = P[e][1], V = P[e][2], D = P[e][3];
                const double p = A + H, m = A - H, r2 = V + D, u = V - D;
                tp[(2 * gi) * TS + 2 * gj] = (p + r2) * 0.5;
                tp[(2 * gi) * TS + 2 * gj + 1] = (p - r2) * 0.5;
                tp[(2 * gi + 1) * TS + 2 * gj] = (m + u) * 0.5;
                tp[(2 * gi + 1) * TS + 2 * gj + 1] = (m - u) * 0.5;
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < s * s * s; i += blockDim.x) {
            const int z = i / (s * s), r = i % (s * s), ii = r / s, jj = r % s;
            x[(z * TS + ii) * TS + jj] = t[(z * TS + ii) * TS + jj];
        }
        __syncthreads();
    }
}

// Device index ((yy*nx + xx)*P + zz) of local cube position (z, i, j) of tile
// (kt, ti, tj), its level and activity (slab-local 3D Mallat layout).
struct CoefInfo3 { uint64_t idx; bool approx; bool active; };
__device__ __forceinline__ CoefInfo3 coef_info3(int z, int i, int j, int kt, int ti, int tj, int L, int nx, int ny,
                                                int nzl, int P, const uint8_t* __restrict__ act, const ActOff& off) {
    CoefInfo3 ci;
    const int m = max(z, max(i, j));
    if (m == 0) {
        ci.idx = ((uint64_t)ti * nx + tj) * P + kt;
        ci.approx = true; ci.active = true;
        return ci;
    }
    const int lg = 31 - __clz(m), l = L - lg, half = 1 << lg;
    const int bk = kt * half + (z & (half - 1)), bi = ti * half + (i & (half - 1)), bj = tj * half + (j & (half - 1));
    const int dl = nzl >> l, hl = ny >> l, wl = nx >> l;
    const int zz = (z >= half ? dl : 0) + bk, yy = (i >= half ? hl : 0) + bi, xx = (j >= half ? wl : 0) + bj;
    ci.idx = ((uint64_t)yy * nx + xx) * P + zz;
    ci.approx = false;
    ci.active = act[off.off[l] + ((uint64_t)bk * hl + bi) * wl + bj] != 0;
    return ci;
}

// One CTA per (TS x TS x TS) tile.  mode 0: synthesis (beta -> mu, mu64);
// mode 1: analysis of g, root solve of active z, synthesis; mode 2: analysis only.
__global__ void k_tile3h(int mode, int nx, int ny, int nzl, int P, int L, const double* __restrict__ g,
                         const double* __restrict__ bm, const double* __restrict__ bdata,
                         const uint8_t* __restrict__ act, ActOff off, float* __restrict__ beta,
                         float* __restrict__ mu, double* __restrict__ mu64, double* __restrict__ out,
                         double* __restrict__ bp_out, double* __restrict__ bm_out, double Z0,
                         unsigned long long* __restrict__ counters, int* __restrict__ flag) {
    extern __shared__ double smh[];
    const int TS = 1 << L, T3 = TS * TS * TS;
    double* x = smh;
    double* t = smh + T3;
    const int tj = blockIdx.x, ti = blockIdx.y, kt = blockIdx.z;
    auto vox = [&](int z, int i, int j) -> uint64_t {
        return ((uint64_t)(ti * TS + i) * nx + (tj * TS + j)) * P + (kt * TS + z);
    };
    if (mode != 0) {
        for (int e = threadIdx.x; e < T3; e += blockDim.x) {  // z fastest: contiguous slab runs
            const int z = e % TS, r = e / TS, i = r / TS, j = r % TS;
            x[(z * TS + i) * TS + j] = g[vox(z, i, j)];
        }
        __syncthreads();
        cube_fwd(x, t, TS, L);
    }
    if (mode == 2) {
        for (int e = threadIdx.x; e < T3; e += blockDim.x) {
            const int z = e % TS, r = e / TS, i = r / TS, j = r % TS;
            const CoefInfo3 ci = coef_info3(z, i, j, kt, ti, tj, L, nx, ny, nzl, P, act, off);
            out[ci.idx] = x[(z * TS + i) * TS + j];
        }
        return;
    }
    if (mode == 3) {   // b+ / b- of every coefficient only (wamgpu_get_stats after a coarse-domain update)
        for (int e = threadIdx.x; e < T3; e += blockDim.x) {
            const int z = e % TS, r = e / TS, i = r / TS, j = r % TS;
            const CoefInfo3 ci = coef_info3(z, i, j, kt, ti, tj, L, nx, ny, nzl, P, act, off);
            const double bmv = ci.approx ? 0.0 : bm[ci.idx];
            bp_out[ci.idx] = x[(z * TS + i) * TS + j] - bmv;
            bm_out[ci.idx] = bmv;
        }
        return;
    }
    unsigned long long upd = 0, deg = 0;
    for (int e = threadIdx.x; e < T3; e += blockDim.x) {
        const int z = e % TS, r = e / TS, i = r / TS, j = r % TS;
        const CoefInfo3 ci = coef_info3(z, i, j, kt, ti, tj, L, nx, ny, nzl, P, act, off);
        float bo = beta[ci.idx];
        if (mode == 1) {
            const double bmv = ci.approx ? 0.0 : bm[ci.idx];
            const double bpv = x[(z * TS + i) * TS + j] - bmv;
            if (bp_out) { bp_out[ci.idx] = bpv; bm_out[ci.idx] = bmv; }
            if (ci.active) {
                double nb;
                const int rr = solve_update(bdata[ci.idx], bpv, bmv, Z0, (double)bo, &nb);
                if (rr == 0) {
                    if (!isfinite(nb)) atomicOr(flag, 4);
                    bo = (float)nb;
                    beta[ci.idx] = bo;
                    ++upd;
                } else if (rr == 2) {
                    ++deg;
                }
            }
        }
        x[(z * TS + i) * TS + j] = (double)bo;
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
    cube_inv(x, t, TS, L);
    for (int e = threadIdx.x; e < T3; e += blockDim.x) {
        const int z = e % TS, r = e / TS, i = r / TS, j = r % TS;
        const uint64_t p = vox(z, i, j);
        mu[p] = (float)x[(z * TS + i) * TS + j];
        if (mu64) mu64[p] = x[(z * TS + i) * TS + j];
    }
}

// k_tile3h mode 1 in the COARSE domain (kernels3c.cuh): while the finest active
// level is k + 1, the update needs only the levels above k, i.e. the leading
// (TS >> k)^3 corner of every tile's transform, and that corner is the transform
// of the 2^k-cube sums G of g.  One CTA per tile works on the (TS >> k)^3 cube:
//   a_k   = G kC3^k 2^-k   (k roundings, exactly what k levels of cube_fwd make of the
//           cube mean G 8^-k spread over the cube: sums of equal values and the
//           factors 1/2, 4 are exact, only the products by kC3 round)
//   cube_fwd over the remaining L - k levels, the same root solves, cube_inv,
//   mu_c = k times (v kC3) / 2   (cube_inv with zero details below level k + 1)
// so beta and the coarse mu are BIT-IDENTICAL to the full-tile update followed by
// k_mu_coarse_z.  The coefficient positions of the corner are the tile's own
// (coef_info3 unchanged).  mu_c goes straight into the z-coarse forward operand;
// the pixel mu is left stale (synthesised from beta when read).  b+ / b- of the
// levels below k + 1 are not produced here (k_tile3h mode 3 on demand).
// gc: Nc*seg rows of Pw doubles, (hi, lo) pairs per z-group (k_back3s over Hc).
__global__ void k_tile3hc(int k, int nx, int ny, int nzl, int P, int L, int Pw, int seg, int Pc,
                          const double* __restrict__ gc, const double* __restrict__ bm,
                          const double* __restrict__ bdata, const uint8_t* __restrict__ act, ActOff off,
                          float* __restrict__ beta, float* __restrict__ muc, double* __restrict__ bp_out,
                          double* __restrict__ bm_out, double Z0, unsigned long long* __restrict__ counters,
                          int* __restrict__ flag) {
    extern __shared__ double smh[];
    const int Lc = L - k, TS = 1 << Lc, T3 = TS * TS * TS, nxc = nx >> k;
    double* x = smh;
    double* t = smh + T3;
    const int tj = blockIdx.x, ti = blockIdx.y, kt = blockIdx.z;
    const double half_k = 1.0 / (double)(1 << k);
    for (int e = threadIdx.x; e < T3; e += blockDim.x) {
        const int z = e % TS, r = e / TS, i = r / TS, j = r % TS;
        const uint64_t B = (uint64_t)(ti * TS + i) * nxc + (tj * TS + j);
        const int zg = kt * TS + z;
        double hi = 0.0, lo = 0.0;
        for (int sg = 0; sg < seg; ++sg) {
            const double2 v = __ldg(reinterpret_cast<const double2*>(gc + (B * seg + sg) * Pw) + zg);
            hi += v.x; lo += v.y;
        }
        double v = hi + lo;
        for (int q = 0; q < k; ++q) v = v * kC3;
        x[(z * TS + i) * TS + j] = v * half_k;
    }
    __syncthreads();
    cube_fwd(x, t, TS, Lc);
    unsigned long long upd = 0, deg = 0;
    for (int e = threadIdx.x; e < T3; e += blockDim.x) {
        const int z = e % TS, r = e / TS, i = r / TS, j = r % TS;
        const CoefInfo3 ci = coef_info3(z, i, j, kt, ti, tj, L, nx, ny, nzl, P, act, off);
        float bo = beta[ci.idx];
        const double bmv = ci.approx ? 0.0 : bm[ci.idx];
        const double bpv = x[(z * TS + i) * TS + j] - bmv;
        if (bp_out) { bp_out[ci.idx] = bpv; bm_out[ci.idx] = bmv; }
        if (ci.active) {
            double nb;
            const int rr = solve_update(bdata[ci.idx], bpv, bmv, Z0, (double)bo, &nb);
            if (rr == 0) {
                if (!isfinite(nb)) atomicOr(flag, 4);
                bo = (float)nb;
                beta[ci.idx] = bo;
                ++upd;
            } else if (rr == 2) {
                ++deg;
            }
        }
        x[(z * TS + i) * TS + j] = (double)bo;
    }
    // (blockDim.x is a multiple of 32: full warps)
    for (int o = 16; o > 0; o >>= 1) {
        upd += __shfl_xor_sync(0xffffffffu, upd, o);
        deg += __shfl_xor_sync(0xffffffffu, deg, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (upd) atomicAdd(counters + 0, upd);
        if (deg) atomicAdd(counters + 1, deg);
    }
    __syncthreads();
    cube_inv(x, t, TS, Lc);
    for (int e = threadIdx.x; e < T3; e += blockDim.x) {
        const int z = e % TS, r = e / TS, i = r / TS, j = r % TS;
        double v = x[(z * TS + i) * TS + j];
        for (int q = 0; q < k; ++q) v = (v * kC3) * 0.5;
        const uint64_t B = (uint64_t)(ti * TS + i) * nxc + (tj * TS + j);
        muc[B * Pc + (kt * TS + z)] = (float)v;
    }
}

// ------------------------------------------ view-group update (RS / AG)
// Exchange buffers in the tile-major chunk layout of TileMap (kernels3d.cuh):
//   T (reduce-scatter): [g of all chunks (Rv*CT) || b- of all chunks (Rv*CT)],
//     written directly by k_back3s / k_split3h_e (tmap.L != 0);
//   U (all-gather every iteration), float chunks of CU = CT + 4: [mu plane
//     (CT) || 2 u64 counts];
//   B: the member's beta plane (CT floats, tile-major), where its tiles' beta
//     lives between iterations.  The planes are all-gathered and scattered to
//     the slab-Mallat beta only at expansions and at the end of each
//     iterate/run call (wamgpu.cu sync_beta), not every iteration.
__host__ __device__ inline uint64_t u_chunk(const TileMap& m) { return m.CT + 4; }

// k_tile3h mode 1 over this member's tiles: inputs from its summed chunks
// (gs = g part, bs = b- part), beta from / to its plane B, mu into its U chunk
__global__ void k_tile3h_own(TileMap tm, int P, int t0, const double* __restrict__ gs,
                             const double* __restrict__ bs, const double* __restrict__ bdata,
                             const uint8_t* __restrict__ act, ActOff off, float* __restrict__ U,
                             float* __restrict__ B,
                             double* __restrict__ bp_out, double* __restrict__ bm_out, double Z0,
                             int* __restrict__ flag) {
    extern __shared__ double smh[];
    const int L = tm.L, TS = 1 << L, T3 = TS * TS * TS;
    double* x = smh;
    double* t = smh + T3;
    const int tj = blockIdx.x, ti = t0 + blockIdx.y, kt = blockIdx.z;
    const uint64_t lt = ((uint64_t)blockIdx.y * tm.TX + tj) * tm.TZ + kt;
    gs += lt * T3;
    bs += lt * T3;
    float* um = U + lt * T3;
    float* ub = B + lt * T3;
    for (int e = threadIdx.x; e < T3; e += blockDim.x) {
        const int z = e % TS, q = e / TS, i = q / TS, j = q % TS;
        x[(z * TS + i) * TS + j] = gs[e];
    }
    __syncthreads();
    cube_fwd(x, t, TS, L);
    unsigned long long upd = 0, deg = 0;
    for (int e = threadIdx.x; e < T3; e += blockDim.x) {
        const int z = e % TS, q = e / TS, i = q / TS, j = q % TS;
        const CoefInfo3 ci = coef_info3(z, i, j, kt, ti, tj, L, tm.nx, tm.ny, tm.nzl, P, act, off);
        float bo = ub[e];
        const double bmv = ci.approx ? 0.0 : bs[e];
        const double bpv = x[(z * TS + i) * TS + j] - bmv;
        if (bp_out) { bp_out[ci.idx] = bpv; bm_out[ci.idx] = bmv; }
        if (ci.active) {
            double nb;
            const int rr = solve_update(bdata[ci.idx], bpv, bmv, Z0, (double)bo, &nb);
            if (rr == 0) {
                if (!isfinite(nb)) atomicOr(flag, 4);
                bo = (float)nb;
                ub[e] = bo;
                ++upd;
            } else if (rr == 2) {
                ++deg;
            }
        }
        x[(z * TS + i) * TS + j] = (double)bo;
    }
    for (int o = 16; o > 0; o >>= 1) {
        upd += __shfl_xor_sync(0xffffffffu, upd, o);
        deg += __shfl_xor_sync(0xffffffffu, deg, o);
    }
    if ((threadIdx.x & 31) == 0) {
        unsigned long long* cnt = reinterpret_cast<unsigned long long*>(U + tm.CT);
        if (upd) atomicAdd(cnt + 0, upd);
        if (deg) atomicAdd(cnt + 1, deg);
    }
    __syncthreads();
    cube_inv(x, t, TS, L);
    for (int e = threadIdx.x; e < T3; e += blockDim.x) {
        const int z = e % TS, q = e / TS, i = q / TS, j = q % TS;
        um[e] = (float)x[(z * TS + i) * TS + j];
    }
}

// every chunk's mu plane -> the voxel slab (grid-stride over elements, z
// fastest on both sides); thread 0 adds the members' counts (rank order)
__global__ void k_unpack_mu(TileMap tm, int P, int members, const float* __restrict__ U, float* __restrict__ mu,
                            unsigned long long* __restrict__ counters) {
    const int TS = 1 << tm.L, T3 = TS * TS * TS;
    const uint64_t CU = u_chunk(tm), n = tm.CT * (uint64_t)members;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = k / tm.CT, w = k % tm.CT, lt = w / T3;
        const int e = (int)(w % T3);
        const int kt = (int)(lt % tm.TZ), tj = (int)((lt / tm.TZ) % tm.TX), ti = (int)(lt / ((uint64_t)tm.TZ * tm.TX)) +
                       (int)r * tm.rows;
        const int z = e % TS, q = e / TS, i = q / TS, j = q % TS;
        mu[((uint64_t)(ti * TS + i) * tm.nx + (tj * TS + j)) * P + (kt * TS + z)] = U[r * CU + w];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long a = 0, b = 0;
        for (int m = 0; m < members; ++m) {
            const unsigned long long* cnt = reinterpret_cast<const unsigned long long*>(U + m * CU + tm.CT);
            a += cnt[0];
            b += cnt[1];
        }
        counters[0] += a;
        counters[1] += b;
    }
}

// beta planes <-> slab Mallat beta.  dir 0: the gathered planes of chunks
// [r0, r0+nchunks) -> beta; dir 1: beta -> the member's own plane (r0 = its
// index, nchunks = 1; at wam_init)
__global__ void k_beta_planes(TileMap tm, int P, int r0, int nchunks, float* __restrict__ planes,
                              float* __restrict__ beta, const uint8_t* __restrict__ act, ActOff off, int dir) {
    const int TS = 1 << tm.L, T3 = TS * TS * TS;
    const uint64_t n = tm.CT * (uint64_t)nchunks;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t rr = k / tm.CT, w = k % tm.CT, lt = w / T3;
        const int r = r0 + (int)rr;
        const int e = (int)(w % T3);
        const int kt = (int)(lt % tm.TZ), tj = (int)((lt / tm.TZ) % tm.TX), ti = (int)(lt / ((uint64_t)tm.TZ * tm.TX)) +
                       r * tm.rows;
        const int z = e % TS, q = e / TS, i = q / TS, j = q % TS;
        const CoefInfo3 ci = coef_info3(z, i, j, kt, ti, tj, tm.L, tm.nx, tm.ny, tm.nzl, P, act, off);
        float* up = planes + rr * tm.CT + w;
        if (dir) *up = beta[ci.idx];
        else beta[ci.idx] = *up;
    }
}

// Expansion criterion of the split update: each member synthesises only its
// own tiles from its beta plane (fp64, the same cube_inv as k_tile3h mode 0,
// so mu64 is bit-identical) into mu64 and one max per tile in part[].
__global__ void k_crit_own(TileMap tm, int P, int t0, const float* __restrict__ B, double* __restrict__ mu64,
                           double* __restrict__ part) {
    extern __shared__ double smh[];
    const int L = tm.L, TS = 1 << L, T3 = TS * TS * TS;
    double* x = smh;
    double* t = smh + T3;
    const int tj = blockIdx.x, ti = t0 + blockIdx.y, kt = blockIdx.z;
    const uint64_t lt = ((uint64_t)blockIdx.y * tm.TX + tj) * tm.TZ + kt;
    const float* ub = B + lt * T3;
    for (int e = threadIdx.x; e < T3; e += blockDim.x) {
        const int z = e % TS, q = e / TS, i = q / TS, j = q % TS;
        x[(z * TS + i) * TS + j] = (double)ub[e];
    }
    __syncthreads();
    cube_inv(x, t, TS, L);
    double m = -DBL_MAX;
    for (int e = threadIdx.x; e < T3; e += blockDim.x) {
        const int z = e % TS, q = e / TS, i = q / TS, j = q % TS;
        const double v = x[(z * TS + i) * TS + j];
        mu64[((uint64_t)(ti * TS + i) * tm.nx + (tj * TS + j)) * P + (kt * TS + z)] = v;
        m = fmax(m, v);
    }
    m = warp_max(m);
    __shared__ double sm[32];
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = -DBL_MAX;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, sm[w]);
        part[lt] = r;
    }
}

// tree bytes <-> doubles (the view group merges its members' marks with a MAX)
__global__ void k_bytes_d(const uint8_t* __restrict__ a, double* __restrict__ d, uint8_t* __restrict__ out,
                          uint64_t n, int dir) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (dir == 0) d[i] = a[i] ? 1.0 : 0.0;
        else out[i] = d[i] > 0.0 ? 1 : 0;
    }
}

// ------------------------------------------------------------ criterion
__global__ void k_max_slab(const double* __restrict__ v, uint64_t n, int nzl, int P, double* __restrict__ part) {
    double m = -DBL_MAX;
    const uint64_t tot = n * (uint64_t)nzl;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (uint64_t)gridDim.x * blockDim.x)
        m = fmax(m, v[(i / nzl) * P + i % nzl]);
    m = warp_max(m);
    __shared__ double s[32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = -DBL_MAX;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, s[w]);
        part[blockIdx.x] = r;
    }
}

// voxel (x, s) with mu > thr activates the coarsest inactive 3D block (OLD tree)
// (voxels e0 .. e1-1 of the slab, e = x*nzl + s: the split update marks only
// its own tile rows)
__global__ void k_mark3h(int nx, int ny, int nzl, int P, int L, const double* __restrict__ mu64, double thr,
                         const uint8_t* __restrict__ act_old, uint8_t* __restrict__ act_new, ActOff off,
                         uint64_t e0, uint64_t e1) {
    const uint64_t e = e0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= e1) return;
    const uint64_t xv = e / nzl;
    const int s = (int)(e % nzl);
    if (!(mu64[xv * P + s] > thr)) return;
    const int iy = (int)(xv / nx), ix = (int)(xv % nx);
    for (int l = L; l >= 1; --l) {
        const uint64_t b = off.off[l] + ((uint64_t)(s >> l) * (ny >> l) + (iy >> l)) * (nx >> l) + (ix >> l);
        if (!act_old[b]) { act_new[b] = 1; return; }
    }
}

// ------------------------------------------------------------ expansion walk
// One warp per level over 32 staged rays (as k_walk_lv).  Tree: anyb bits (one
// per (l, in-plane block)) in shared memory; per-block z-bit words in global
// (W_l words per block, bit k = z-block k of the slab).
// MODE 1: Z(y) = max_s [zA(y) + tot_L(k_L(s)) + ... + tot_1(k_1(s))] with
//   tot_l(k) = sum over (ray-order) level-l blocks b with (k, b) active of
//   t = |Hl|+|Vl|+|Dl|+|Ah|+|Hh|+|Vh|+|Dh| (each psi c^l) — oracle z_row3;
//   cnt[y*L + l-1] = number of level-l blocks b crossed with any active k.
// MODE 2: emit one Psi entry per such (y, b): key = koff[l] + b, payload at pos.
template <int MODE, int L>
__global__ void __launch_bounds__(32 * 6) k_walk3h(uint64_t M, const unsigned long long* __restrict__ rp,
                                                   const uint2* __restrict__ A, int nx, int ny, int nzl,
                                                   const unsigned* __restrict__ tbits, ActOff boff, int tree_words,
                                                   const unsigned* __restrict__ zbits, ActOff zoff, ActOff koff,
                                                   const double* __restrict__ zA, double* __restrict__ zrow,
                                                   unsigned long long* __restrict__ cnt,
                                                   const unsigned long long* __restrict__ pos,
                                                   unsigned* __restrict__ keys, uint2* __restrict__ vidx,
                                                   unsigned* __restrict__ pray, float4* __restrict__ ppsi,
                                                   int split1) {
    // The tree bits stay in global memory (read-only, L1-resident: 43 KB at cfg4).
    // Holding them in shared memory, as the first version did, left 2 CTAs --
    // 2 to 12 warps -- per SM (82 KB per CTA at cfg4), and the walk ran at 2% of
    // the HBM roofline on latency alone.
    extern __shared__ unsigned char dsm[];
    double* stot = reinterpret_cast<double*>(dsm);   // MODE 1: sum over the walked levels of (nzl>>l)*32
    (void)tree_words;
    __shared__ uint2 buf[32][33];
    __shared__ unsigned long long s_lo[32], s_len[32];
    // split1 (MODE 1, level 1 walked): one extra warp also walks level 1 and
    // owns the high 16 bits of every z-bit word, the level-1 warp the low 16,
    // so the heaviest flush loop is shared (each tot slot keeps one owner and
    // its ray-order sum)
    const int nwarp = blockDim.x >> 5, nlev = nwarp - split1;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, l = w < nlev ? L - w : 1;
    const unsigned hmask = !split1 || l != 1 ? 0xffffffffu : (w < nlev ? 0x0000ffffu : 0xffff0000u);
    int toff = 0;  // offset of this level's tot block in stot
    for (int k = L; k > l; --k) toff += (nzl >> k) * 32;
    const int nk = nzl >> l;
    if (MODE == 1)
        for (int i = lane; i < nk * 32; i += 32) stot[toff + i] = 0.0;
    const uint64_t y = (uint64_t)blockIdx.x * 32 + lane;
    if (w == 0) {
        uint64_t lo = 0, hi = 0;
        if (y < M) { lo = rp[y]; hi = rp[y + 1]; }
        s_lo[lane] = lo;
        s_len[lane] = hi - lo;
    }
    __syncthreads();
    unsigned long long maxlen = s_len[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
    const unsigned long long len = s_len[lane];
    const bool pow2 = (nx & (nx - 1)) == 0;
    const int lgx = 31 - __clz(nx);
    const int wl = nx >> l;
    const unsigned bo = (unsigned)boff.off[l];
    const double sc = 1.0 / (double)(1 << l), cl = cpow3(l);
    const int W = (nk + 31) >> 5;

    int cur = -1, cq = -1;
    bool av = false;
    double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0, qa = 0.0;
    unsigned long long count = 0, wp = 0;
    if (MODE == 2 && y < M) wp = pos[y * L + (l - 1)];

    auto park = [&]() {
        q0 = cq == 0 ? qa : q0;
        q1 = cq == 1 ? qa : q1;
        q2 = cq == 2 ? qa : q2;
        q3 = cq == 3 ? qa : q3;
    };
    auto flush = [&]() {
        if (av) {
            park();
            const double st = q0 + q1, sb = q2 + q3;
            const double pA = (st + sb) * sc, pH = (st - sb) * sc, pV = ((q0 + q2) - (q1 + q3)) * sc,
                         pD = ((q0 + q3) - (q1 + q2)) * sc;
            if (MODE == 1) {
                const double hh = fabs(pH * cl), vv = fabs(pV * cl), dd = fabs(pD * cl), aa = fabs(pA * cl);
                const double t = (((((hh + vv) + dd) + aa) + hh) + vv) + dd;
                const unsigned* zb = zbits + zoff.off[l] + (uint64_t)cur * W;
                // four set z-blocks per step: their tot slots are distinct, so
                // the four load-add-store chains overlap (the level-1 warp's
                // per-flush loop is what the other level warps wait for at the
                // round barrier, profiles/r04_ncu_walk_src.txt); each slot still
                // receives t in ray order, so the sums are unchanged
                double* sb = stot + toff + lane;
                for (int wi = 0; wi < W; ++wi) {
                    unsigned m = zb[wi] & hmask;
                    while (m) {
                        const int k0 = __ffs(m) - 1;
                        m &= m - 1;
                        const int k1 = m ? __ffs(m) - 1 : -1;
                        m &= m - 1;
                        const int k2 = m ? __ffs(m) - 1 : -1;
                        m &= m - 1;
                        const int k3 = m ? __ffs(m) - 1 : -1;
                        m &= m - 1;
                        double* p0 = sb + (wi * 32 + k0) * 32;
                        double* p1 = sb + (wi * 32 + (k1 < 0 ? k0 : k1)) * 32;
                        double* p2 = sb + (wi * 32 + (k2 < 0 ? k0 : k2)) * 32;
                        double* p3 = sb + (wi * 32 + (k3 < 0 ? k0 : k3)) * 32;
                        const double v0 = *p0, v1 = *p1, v2 = *p2, v3 = *p3;
                        *p0 = v0 + t;
                        if (k1 >= 0) *p1 = v1 + t;
                        if (k2 >= 0) *p2 = v2 + t;
                        if (k3 >= 0) *p3 = v3 + t;
                    }
                }
                ++count;
            } else {
                keys[wp] = (unsigned)(koff.off[l] + cur);
                vidx[wp] = make_uint2((unsigned)wp, 0u);
                pray[wp] = (unsigned)y;
                ppsi[wp] = make_float4((float)pA, (float)pH, (float)pV, (float)pD);
                ++wp;
            }
            q0 = q1 = q2 = q3 = 0.0;
        }
        cq = -1;
        qa = 0.0;
    };

    for (unsigned long long base = 0; base < maxlen; base += 32) {
        for (int j = w; j < 32; j += nwarp) {
            const unsigned long long nj = s_len[j];
            const bool ok = base + lane < nj;
            cp_async8(&buf[j][lane], A + (ok ? s_lo[j] + base + lane : 0), ok);
        }
        cp_async_wait_all();
        __syncthreads();
        const int n = (int)min(32ull, len > base ? len - base : 0ull);
        for (int i = 0; i < n; ++i) {
            const uint2 e = buf[lane][i];
            int ix, iy;
            if (pow2) { ix = (int)(e.x & (unsigned)(nx - 1)); iy = (int)(e.x >> lgx); }
            else { iy = (int)(e.x / (unsigned)nx); ix = (int)(e.x % (unsigned)nx); }
            const int key = (iy >> l) * wl + (ix >> l);
            if (key != cur) {
                flush();
                cur = key;
                const unsigned bit = bo + (unsigned)key;
                av = (__ldg(tbits + (bit >> 5)) >> (bit & 31)) & 1u;
            }
            if (av) {
                const int quad = (((iy >> (l - 1)) & 1) << 1) | ((ix >> (l - 1)) & 1);
                if (quad != cq) {
                    if (cq >= 0) park();
                    cq = quad;
                    qa = 0.0;
                }
                qa += hval(e);
            }
        }
        __syncthreads();
    }
    flush();
    if (MODE == 1) {
        if (y < M && w < nlev) cnt[y * L + (l - 1)] = count;
        __syncthreads();
        if (w == 0 && y < M) {
            for (int k = 1; k <= L - nlev; ++k) cnt[y * L + (k - 1)] = 0;
            double best = 0.0;
            for (int s = 0; s < nzl; ++s) {
                double z = zA[y];
                int o = 0;
                for (int k = L; k >= 1; --k) {
                    if (k > L - nlev) z += stot[o + (s >> k) * 32 + lane];
                    o += (nzl >> k) * 32;
                }
                best = fmax(best, z);
            }
            zrow[y] = best;
        }
    }
}

// Payload gather after the key sort: E3 entries in (key, ray-insertion) order.
__global__ void k_gather_psi(uint64_t n, const uint2* __restrict__ sidx, const unsigned* __restrict__ pray,
                             const float4* __restrict__ ppsi, unsigned* __restrict__ eray,
                             float4* __restrict__ epsi) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned j = sidx[i].x;
    eray[i] = pray[j];
    epsi[i] = ppsi[j];
}

// ------------------------------------------------------------ split (3D)
// Warp per (level l, in-plane block b) with any active z-block: over its Psi
// list, lanes own SPL slices; per entry the negative-part multipliers are
//   z-low p in H,V,D:    m_lo = m_hi = min(psi_p c^l, 0)
//   z-high p in A,H,V,D: m_lo = min(psi_p c^l, 0), m_hi = -max(psi_p c^l, 0)
// and slice s (z-block k = s>>l, half (s>>(l-1))&1) adds m_half * q(y, s).
// Consecutive slice pairs (2m, 2m+1) share a half for l >= 2 (one fma on
// q0+q1) and split one block's halves for l == 1.  Pair partials are summed
// over each block's slices (ascending) and written for the active (k, b).
template <int SPL>
__global__ void __launch_bounds__(128) k_split3h(uint64_t nlist, const uint2* __restrict__ list, int nx, int ny,
                                                 int nzl, const unsigned long long* __restrict__ ptr,
                                                 const unsigned* __restrict__ eray, const float4* __restrict__ epsi,
                                                 const float* __restrict__ q, const uint8_t* __restrict__ act,
                                                 ActOff off, ActOff koff, double* __restrict__ bm, TileMap tmap) {
    using V = typename SlabVec<SPL>::T;
    constexpr int P = 32 * SPL;
    constexpr int NG = SPL >= 2 ? SPL / 2 : 1;   // slice groups per lane (pairs, or the single slice)
    __shared__ double red[4][7][32 * NG];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t it = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < nlist; it += W) {
        const unsigned b = list[it].x;
        const int l = (int)list[it].y;
        const double cl = cpow3(l);
        const uint64_t key = koff.off[l] + b;
        // half of each of this lane's slices (SPL == 1: the single slice)
        bool hi1 = false;
        if (SPL == 1) hi1 = ((lane >> (l - 1)) & 1) != 0;
        double acc[NG][7];
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
            for (int t = 0; t < 7; ++t) acc[g][t] = 0.0;
        constexpr int U = 4;
        const uint64_t e0 = ptr[key], e1 = ptr[key + 1];
        for (uint64_t e = e0; e < e1; e += U) {
            unsigned yv[U];
            float4 ps[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool ok = e + u < e1;
                const uint64_t ei = ok ? e + u : e;   // always a valid index
                yv[u] = __ldg(eray + ei);
                ps[u] = __ldg(epsi + ei);
                if (!ok) ps[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            V qv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) qv[u] = __ldg(reinterpret_cast<const V*>(q + (uint64_t)yv[u] * P) + lane);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const double pA = (double)ps[u].x * cl, pH = (double)ps[u].y * cl, pV = (double)ps[u].z * cl,
                             pD = (double)ps[u].w * cl;
                const double lowm[3] = {fmin(pH, 0.0), fmin(pV, 0.0), fmin(pD, 0.0)};
                const double hp[4] = {pA, pH, pV, pD};
                double mlo[4], mhi[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) { mlo[t] = fmin(hp[t], 0.0); mhi[t] = -fmax(hp[t], 0.0); }
                float f[SPL];
                unpack(qv[u], f);
                if constexpr (SPL == 1) {
                    const double qq = (double)f[0];
#pragma unroll
                    for (int t = 0; t < 3; ++t) acc[0][t] = fma(lowm[t], qq, acc[0][t]);
#pragma unroll
                    for (int t = 0; t < 4; ++t) acc[0][3 + t] = fma(hi1 ? mhi[t] : mlo[t], qq, acc[0][3 + t]);
                } else {
                  if (l >= 2) {
#pragma unroll
                    for (int g = 0; g < NG; ++g) {
                        const int s = lane * SPL + 2 * g;
                        const bool hh = ((s >> (l - 1)) & 1) != 0;
                        const double qq = (double)f[2 * g] + (double)f[2 * g + 1];
#pragma unroll
                        for (int t = 0; t < 3; ++t) acc[g][t] = fma(lowm[t], qq, acc[g][t]);
#pragma unroll
                        for (int t = 0; t < 4; ++t) acc[g][3 + t] = fma(hh ? mhi[t] : mlo[t], qq, acc[g][3 + t]);
                    }
                } else {  // l == 1: the pair is one z-block, slice 2g its low half, 2g+1 its high half
#pragma unroll
                    for (int g = 0; g < NG; ++g) {
                        const double q0 = (double)f[2 * g], q1 = (double)f[2 * g + 1], qq = q0 + q1;
#pragma unroll
                        for (int t = 0; t < 3; ++t) acc[g][t] = fma(lowm[t], qq, acc[g][t]);
#pragma unroll
                        for (int t = 0; t < 4; ++t) acc[g][3 + t] = fma(mhi[t], q1, fma(mlo[t], q0, acc[g][3 + t]));
                    }
                  }
                }
            }
        }
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
            for (int t = 0; t < 7; ++t) red[wib][t][lane * NG + g] = acc[g][t];
        __syncwarp();
        const int nk = nzl >> l, hl = ny >> l, wl = nx >> l, dl = nk;
        const int bi = (int)(b / wl), bj = (int)(b % wl);
        const int gper = SPL == 1 ? 1 : 2;   // slices per group
        for (int k = lane; k < nk; k += 32) {
            if (!act[off.off[l] + ((uint64_t)k * hl + bi) * wl + bj]) continue;
            const int zz[7] = {k, k, k, dl + k, dl + k, dl + k, dl + k};
            const int yy[7] = {hl + bi, bi, hl + bi, bi, hl + bi, bi, hl + bi};
            const int xx[7] = {bj, wl + bj, wl + bj, bj, bj, wl + bj, wl + bj};
            const int g0 = (k << l) / gper, g1 = ((k + 1) << l) / gper;
#pragma unroll
            for (int t = 0; t < 7; ++t) {
                double sum = 0.0;
                for (int gg = g0; gg < g1; ++gg) sum += red[wib][t][gg];
                bm[tmap.L ? coef_tile_pos(tmap, l, yy[t], xx[t], zz[t]) : ((uint64_t)yy[t] * nx + xx[t]) * P + zz[t]] =
                    sum;
            }
        }
        __syncwarp();
    }
}

// k_split3h with E Psi entries in flight per warp: 32/E lanes per entry, each
// lane owning S = SPL*E consecutive slices (S/2 slice pairs).  The per-entry
// multipliers are computed by 32/E lanes instead of 32 (fp64 work per slice
// roughly halves at E = 4); the E entry groups' partials are combined by a
// fixed xor butterfly, then per-block sums as in k_split3h.
// U rounds of E entries: the q rows of round r+1 are loaded before round r is
// consumed (software pipeline; ncu at cfg4 showed 44% of the stall samples on
// the first use of the q gathers with only the current round in flight).
// (A two-stage pipeline -- entries of round r+2 and q rows of round r+1 in flight,
// evict-first Psi loads -- was measured slower: cfg3 9.06 vs 7.82, cfg4 60.3 vs
// 53.9 ms per launch at a 128-register cap, profiles/r06/split_prefetch_ab.txt.)
// Templated on the slab stride P (8 .. 128): S = P*E/32 slices per lane.
template <int P, int E, int U = 2>
__global__ void __launch_bounds__(128) k_split3h_e(uint64_t nlist, const uint2* __restrict__ list, int nx, int ny,
                                                   int nzl, const unsigned long long* __restrict__ ptr,
                                                   const unsigned* __restrict__ eray, const float4* __restrict__ epsi,
                                                   const float* __restrict__ q, const uint8_t* __restrict__ act,
                                                   ActOff off, ActOff koff, double* __restrict__ bm,
                                                   TileMap tmap, const unsigned long long* __restrict__ bptr,
                                                   int B, int band) {
    constexpr int LPE = 32 / E, S = P * E / 32, NG = S / 2;
    static_assert(S >= 2 && S % 4 == 0, "slices per lane: a multiple of 4");
    __shared__ double red[4][7][P / 2];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, grp = lane / LPE, j = lane % LPE;
    const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t it = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < nlist; it += W) {
        const unsigned b = list[it].x;
        const int l = (int)list[it].y;
        const double cl = cpow3(l);
        const uint64_t key = koff.off[l] + b;
        double acc[NG][7];
#pragma unroll
        for (int g = 0; g < NG; ++g)
#pragma unroll
            for (int t = 0; t < 7; ++t) acc[g][t] = 0.0;
        // banded (bptr != nullptr): this launch takes the key's entries whose
        // rays lie in ray band `band` and ADDS their sums to what the earlier
        // bands left in bm (fixed band order: deterministic)
        const uint64_t e0 = bptr ? bptr[key * (uint64_t)(B + 1) + band] : ptr[key];
        const uint64_t e1 = bptr ? bptr[key * (uint64_t)(B + 1) + band + 1] : ptr[key + 1];
        if (band > 0 && e0 == e1) continue;   // nothing to add (uniform over the warp)
        unsigned yv[U];
        float4 ps[U];
        float4 qv[U][S / 4];
        auto load = [&](uint64_t e) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint64_t ee = e + grp + (uint64_t)E * u;
                const bool ok = ee < e1;
                const uint64_t ei = ok ? ee : e0;   // always a valid index
                yv[u] = __ldg(eray + ei);
                ps[u] = ok ? __ldg(epsi + ei) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int v = 0; v < S / 4; ++v)
                    qv[u][v] = __ldg(reinterpret_cast<const float4*>(q + (uint64_t)yv[u] * P + j * S) + v);
        };
        if (e0 < e1) load(e0);
        for (uint64_t e = e0; e < e1; e += (uint64_t)E * U) {
            float4 pc[U];
            float4 qc[U][S / 4];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                pc[u] = ps[u];
#pragma unroll
                for (int v = 0; v < S / 4; ++v) qc[u][v] = qv[u][v];
            }
            if (e + (uint64_t)E * U < e1) load(e + (uint64_t)E * U);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const double pA = (double)pc[u].x * cl, pH = (double)pc[u].y * cl, pV = (double)pc[u].z * cl,
                             pD = (double)pc[u].w * cl;
                const double lowm[3] = {fmin(pH, 0.0), fmin(pV, 0.0), fmin(pD, 0.0)};
                const double hp[4] = {pA, pH, pV, pD};
                double mlo[4], mhi[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) { mlo[t] = fmin(hp[t], 0.0); mhi[t] = -fmax(hp[t], 0.0); }
                float f[S];
#pragma unroll
                for (int v = 0; v < S / 4; ++v) {
                    f[4 * v] = qc[u][v].x; f[4 * v + 1] = qc[u][v].y; f[4 * v + 2] = qc[u][v].z; f[4 * v + 3] = qc[u][v].w;
                }
                if (l >= 2) {
#pragma unroll
                    for (int g = 0; g < NG; ++g) {
                        const int sl = j * S + 2 * g;
                        const bool hh = ((sl >> (l - 1)) & 1) != 0;
                        const double qq = (double)f[2 * g] + (double)f[2 * g + 1];
#pragma unroll
                        for (int t = 0; t < 3; ++t) acc[g][t] = fma(lowm[t], qq, acc[g][t]);
#pragma unroll
                        for (int t = 0; t < 4; ++t) acc[g][3 + t] = fma(hh ? mhi[t] : mlo[t], qq, acc[g][3 + t]);
                    }
                } else {   // l == 1: a pair is one z-block (low half, high half)
#pragma unroll
                    for (int g = 0; g < NG; ++g) {
                        const double q0 = (double)f[2 * g], q1 = (double)f[2 * g + 1], qq = q0 + q1;
#pragma unroll
                        for (int t = 0; t < 3; ++t) acc[g][t] = fma(lowm[t], qq, acc[g][t]);
#pragma unroll
                        for (int t = 0; t < 4; ++t) acc[g][3 + t] = fma(mhi[t], q1, fma(mlo[t], q0, acc[g][3 + t]));
                    }
                }
            }
        }
        // combine the E entry groups (same slices: lanes j, j+LPE, ...), fixed order
#pragma unroll
        for (int o = LPE; o < 32; o <<= 1)
#pragma unroll
            for (int g = 0; g < NG; ++g)
#pragma unroll
                for (int t = 0; t < 7; ++t) acc[g][t] += __shfl_xor_sync(0xffffffffu, acc[g][t], o);
        if (grp == 0) {
#pragma unroll
            for (int g = 0; g < NG; ++g)
#pragma unroll
                for (int t = 0; t < 7; ++t) red[wib][t][j * NG + g] = acc[g][t];
        }
        __syncwarp();
        const int nk = nzl >> l, hl = ny >> l, wl = nx >> l, dl = nk;
        const int bi = (int)(b / wl), bj = (int)(b % wl);
        for (int k = lane; k < nk; k += 32) {
            if (!act[off.off[l] + ((uint64_t)k * hl + bi) * wl + bj]) continue;
            const int zz[7] = {k, k, k, dl + k, dl + k, dl + k, dl + k};
            const int yy[7] = {hl + bi, bi, hl + bi, bi, hl + bi, bi, hl + bi};
            const int xx[7] = {bj, wl + bj, wl + bj, bj, bj, wl + bj, wl + bj};
            const int g0 = (k << l) / 2, g1 = ((k + 1) << l) / 2;
#pragma unroll
            for (int t = 0; t < 7; ++t) {
                double sum = 0.0;
                for (int gg = g0; gg < g1; ++gg) sum += red[wib][t][gg];
                double* o = bm + (tmap.L ? coef_tile_pos(tmap, l, yy[t], xx[t], zz[t])
                                         : ((uint64_t)yy[t] * nx + xx[t]) * P + zz[t]);
                *o = band > 0 ? *o + sum : sum;
            }
        }
        __syncwarp();
    }
}

// ---- split, pipelined (default): k_split3p ---------------------------------
// Same lane map as k_split3h_e (E entry groups of LPE = 32/E lanes, S = P*E/32
// consecutive slices per lane) with the per-entry work cut down.  ncu of
// k_split3h_e at cfg4 (profiles/r06/ncu_split_cfg4_src.txt): DFMA was 12.5% of
// the issue samples; register copies of the software pipeline 20%, fp64
// min/max/select chains for the multipliers 10%, address arithmetic 15%.
//  * sums of q first: qlo / qhi = slice-order sums of the z-block's halves (the
//    SPEC's per-half formulation), then 3 + 4 (+4) FMAs per z-block instead of
//    7 per slice pair; the loop is specialised per level, so which half a slice
//    belongs to is static (no per-pair selects);
//  * c^l is factored out of the sums (one multiplication per output), so the
//    multipliers are plain conversions of min(psi, 0) / min(-psi, 0) taken in
//    fp32 (FMNMX) instead of fp64 compare/select chains after psi * c^l;
//  * q >= 0 moves into fp64 by ONE multiply (f2d_scaled<false>, exact);
//  * level whose half fits a lane (TRICK): z-high = L - Pq with
//    L = sum min(p,0) (qlo+qhi)  (the z-low sum, needed anyway) and
//    Pq = sum p qhi, since min(p,0) qlo - max(p,0) qhi = min(p,0)(qlo+qhi) - p qhi:
//    3 + 3 + 2 FMAs per z-block instead of 3 + 8;
//  * three-stage pipeline on two register sets without copies: (ray, psi) of
//    round r+2 and the q row of round r+1 are in flight while round r is consumed.
// Sums are fp64 FMAs of exact fp32 x fp32 products in entry order per group,
// groups combined by a fixed xor butterfly: deterministic, and within 1e-15
// relative of k_split3h_e (different association; tests compare both to the oracle).
template <int S>
struct SplitSet {
    unsigned y;
    float4 ps;
    float4 q[S / 4];
};
template <int P, int E, int LV, bool TRICK>
__device__ __forceinline__ void split3p_block(unsigned b, int l, int lane, int wib, int nx, int ny, int nzl,
                                              uint64_t e0, uint64_t e1, const unsigned* __restrict__ eray,
                                              const float4* __restrict__ epsi, const float* __restrict__ q,
                                              const uint8_t* __restrict__ act, const ActOff& off,
                                              double* __restrict__ bm, const TileMap& tmap,
                                              double (&red)[4][7][P / 2]) {
    constexpr int LPE = 32 / E, S = P * E / 32;
    static_assert(S == 4 || S == 8, "slices per lane");
    // LV > 0: half size HS = 2^(LV-1) < S, NZ complete z-blocks per lane.
    // LV == 0: runtime level with HS >= S (the lane lies inside one half).
    constexpr int HS = LV > 0 ? (1 << (LV - 1)) : S;
    constexpr int NZ = LV > 0 ? S / (2 * HS) : 1;
    static_assert(LV == 0 || 2 * HS <= S, "level does not fit a lane");
    constexpr int NA = LV > 0 ? 7 * NZ : 7;
    const int grp = lane / LPE, j = lane % LPE;
    const bool hh = LV == 0 ? (((j * S) >> (l - 1)) & 1) != 0 : false;
    double acc[NA];
#pragma unroll
    for (int i = 0; i < NA; ++i) acc[i] = 0.0;
    SplitSet<S> A, B;
    const uint64_t n = e1 - e0;
    const uint64_t nr = (n + E - 1) / E;
    auto load_idx = [&](SplitSet<S>& x, uint64_t r) {
        const uint64_t ee = e0 + r * E + grp;
        const bool ok = ee < e1;
        const uint64_t ei = ok ? ee : e0;   // always a valid index
        x.y = __ldg(eray + ei);
        x.ps = ok ? __ldg(epsi + ei) : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    auto load_q = [&](SplitSet<S>& x) {
        const float4* row = reinterpret_cast<const float4*>(q + (uint64_t)x.y * P + j * S);
#pragma unroll
        for (int v = 0; v < S / 4; ++v) x.q[v] = __ldg(row + v);
    };
    auto step = [&](SplitSet<S>& X, SplitSet<S>& Y, uint64_t r) {
        const float pf[4] = {X.ps.x, X.ps.y, X.ps.z, X.ps.w};
        double m[8];
        if constexpr (LV > 0) {
            // m[0..3] = min(psi_t, 0) (t = A,H,V,D); m[4] = min(-psi_A, 0);
            // m[5..7] = TRICK ? psi_t : min(-psi_t, 0) (t = H,V,D)
#pragma unroll
            for (int t = 0; t < 4; ++t) m[t] = (double)fminf(pf[t], 0.f);
            m[4] = (double)fminf(-pf[0], 0.f);
#pragma unroll
            for (int t = 1; t < 4; ++t) m[4 + t] = TRICK ? (double)pf[t] : (double)fminf(-pf[t], 0.f);
        } else {
            // m[0..2] = min(psi_t, 0) (t = H,V,D: z-low); m[3..6] = this lane's half of z-high
            // (low half min(psi,0), high half min(-psi,0)), scaled by 2^-896 (bit move)
#pragma unroll
            for (int t = 1; t < 4; ++t) m[t - 1] = f2d_scaled<true>(fminf(pf[t], 0.f));
#pragma unroll
            for (int t = 0; t < 4; ++t) m[3 + t] = f2d_scaled<true>(fminf(hh ? -pf[t] : pf[t], 0.f));
        }
        if (r + 2 < nr) load_idx(X, r + 2);
        if (r + 1 < nr) load_q(Y);
        float f[S];
#pragma unroll
        for (int v = 0; v < S / 4; ++v) {
            f[4 * v] = X.q[v].x; f[4 * v + 1] = X.q[v].y; f[4 * v + 2] = X.q[v].z; f[4 * v + 3] = X.q[v].w;
        }
        if constexpr (LV > 0) {
#pragma unroll
            for (int z = 0; z < NZ; ++z) {
                double qlo = f2d_scaled<false>(f[z * 2 * HS]), qhi = f2d_scaled<false>(f[z * 2 * HS + HS]);
#pragma unroll
                for (int i = 1; i < HS; ++i) {
                    qlo += f2d_scaled<false>(f[z * 2 * HS + i]);
                    qhi += f2d_scaled<false>(f[z * 2 * HS + HS + i]);
                }
                const double qall = qlo + qhi;
                double* a = acc + 7 * z;
#pragma unroll
                for (int t = 0; t < 3; ++t) a[t] = fma(m[1 + t], qall, a[t]);
                a[3] = fma(m[4], qhi, fma(m[0], qlo, a[3]));
#pragma unroll
                for (int t = 0; t < 3; ++t) {
                    if constexpr (TRICK) a[4 + t] = fma(m[5 + t], qhi, a[4 + t]);
                    else a[4 + t] = fma(m[5 + t], qhi, fma(m[1 + t], qlo, a[4 + t]));
                }
            }
        } else {
            double qs = f2d_scaled<false>(f[0]);
#pragma unroll
            for (int i = 1; i < S; ++i) qs += f2d_scaled<false>(f[i]);
            qs *= kTwo896;   // exact: the multipliers carry the 2^-896 here
#pragma unroll
            for (int t = 0; t < 7; ++t) acc[t] = fma(m[t], qs, acc[t]);
        }
    };
    if (nr > 0) {
        load_idx(A, 0);
        if (nr > 1) load_idx(B, 1);
        load_q(A);
        for (uint64_t r = 0; r < nr; r += 2) {
            step(A, B, r);
            if (r + 1 < nr) step(B, A, r + 1);
        }
    }
    if constexpr (LV > 0 && TRICK) {
#pragma unroll
        for (int z = 0; z < NZ; ++z)
#pragma unroll
            for (int t = 0; t < 3; ++t) acc[7 * z + 4 + t] = acc[7 * z + t] - acc[7 * z + 4 + t];
    }
    // combine the E entry groups (same slices: lanes j, j+LPE, ...), fixed order
#pragma unroll
    for (int o = LPE; o < 32; o <<= 1)
#pragma unroll
        for (int i = 0; i < NA; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
    // red[t][slot]: t = 0..2 z-low H,V,D; 3..6 z-high A,H,V,D
    if (grp == 0) {
        if constexpr (LV > 0) {
#pragma unroll
            for (int z = 0; z < NZ; ++z)
#pragma unroll
                for (int t = 0; t < 7; ++t) red[wib][t][j * NZ + z] = acc[7 * z + t];
        } else {
#pragma unroll
            for (int t = 0; t < 7; ++t) red[wib][t][j] = acc[t];
        }
    }
    __syncwarp();
    const double cls = cpow3(l) * kTwo896;
    const int nk = nzl >> l, hl = ny >> l, wl = nx >> l, dl = nk;
    const int bi = (int)(b / wl), bj = (int)(b % wl);
    const int per = LV > 0 ? 1 : ((1 << l) / S);   // red slots per z-block
    for (int k = lane; k < nk; k += 32) {
        if (!act[off.off[l] + ((uint64_t)k * hl + bi) * wl + bj]) continue;
        const int zz[7] = {k, k, k, dl + k, dl + k, dl + k, dl + k};
        const int yy[7] = {hl + bi, bi, hl + bi, bi, hl + bi, bi, hl + bi};
        const int xx[7] = {bj, wl + bj, wl + bj, bj, bj, wl + bj, wl + bj};
#pragma unroll
        for (int t = 0; t < 7; ++t) {
            double sum = red[wib][t][k * per];
            for (int gg = 1; gg < per; ++gg) sum += red[wib][t][k * per + gg];
            bm[tmap.L ? coef_tile_pos(tmap, l, yy[t], xx[t], zz[t]) : ((uint64_t)yy[t] * nx + xx[t]) * P + zz[t]] =
                sum * cls;
        }
    }
    __syncwarp();
}
template <int P, int E, bool TRICK, int MINB = 1>
__global__ void __launch_bounds__(128, MINB) k_split3p(uint64_t nlist, const uint2* __restrict__ list, int nx, int ny,
                                                 int nzl, const unsigned long long* __restrict__ ptr,
                                                 const unsigned* __restrict__ eray, const float4* __restrict__ epsi,
                                                 const float* __restrict__ q, const uint8_t* __restrict__ act,
                                                 ActOff off, ActOff koff, double* __restrict__ bm, TileMap tmap) {
    constexpr int S = P * E / 32;
    __shared__ double red[4][7][P / 2];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t it = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < nlist; it += W) {
        const unsigned b = list[it].x;
        const int l = (int)list[it].y;
        const uint64_t key = koff.off[l] + b;
        const uint64_t e0 = ptr[key], e1 = ptr[key + 1];
#define SP(LVv) split3p_block<P, E, LVv, TRICK>(b, l, lane, wib, nx, ny, nzl, e0, e1, eray, epsi, q, act, off, bm, tmap, red)
        if (l == 1) SP(1);
        else if (l == 2) SP(2);
        else if (S == 8 && l == 3) { if constexpr (S == 8) SP(3); }
        else SP(0);
#undef SP
    }
}

// ---- split, CTA per block with a cp.async ring (k_split3c) -------------------
// k_split3p is bound by memory latency, not by instructions: with 12-16 warps
// per SM and one q row (P*4 bytes) per entry in flight per entry group, about
// 12-16 KB per SM are in flight, which by Little's law caps the gathers near
// 2-4 TB/s whatever the instruction count (cfg4: 7.6e9 entries/s x 512 B).  Here
//  * the q rows travel by cp.async into a per-warp ring of D rounds in shared
//    memory (no registers held by loads in flight); each lane copies and later
//    reads back only its own S slices, so no barrier is needed between the two;
//  * (ray, psi) are read 32 entries at a time, coalesced, one entry per lane,
//    into a double-buffered per-warp index buffer (instead of every lane of a
//    group loading its group's entry each round);
//  * WPI warps share one block: each takes a contiguous range of the block's
//    entries, so only 1/WPI as many blocks are in flight and, with the list in
//    Morton order, their rays' q rows stay L2-resident.  The warps' partial
//    sums meet in shared memory in warp order (deterministic).
// Per-entry arithmetic = split3p (per-half sums, c^l factored out, L - Pq).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
// f2d_scaled by ONE 32x32->64 multiply by 2^29 (IMAD.WIDE: lo = u << 29, hi = u >> 3;
// signed: the sign-extending multiply leaves ssss in hi[31:28], one AND keeps s at
// bit 31).  Slower than the shifts in the slab SpMM (kernels3d.cuh) but faster here,
// where the ALU pipe carries the min/select work: cfg4 split 1595 vs 2095 ms per run
// with k_split3p (profiles/r07/ab1.txt, ab2.txt).
template <bool SIGNED>
__device__ __forceinline__ double f2d_wide(float f) {
    if constexpr (SIGNED) {
        long long w;   // inline PTX: nvcc strength-reduces the C++ multiply into shifts again
        asm("mul.wide.s32 %0, %1, 536870912;" : "=l"(w) : "r"(__float_as_int(f)));
        return __hiloint2double((int)(w >> 32) & (int)0x8fffffff, (int)(unsigned)w);
    } else {
        unsigned long long w;
        asm("mul.wide.u32 %0, %1, 536870912;" : "=l"(w) : "r"(__float_as_uint(f)));
        return __longlong_as_double((long long)w);
    }
}
// One entry's contribution for a lane that holds V = S/4 chunks of 4 consecutive
// slices (chunk v starts at slice 4*LPE*v + 4*j: every cp.async / load instruction
// of a group then covers one contiguous run of the q row, whole 32-byte sectors;
// 8 consecutive slices per lane made every sector travel twice, and the split is
// bound by L2 -> SM traffic: ncu lts throughput 80%, profiles/r07/ncu_split3c_cfg4.txt).
// LV 1: two z-blocks per chunk (pairs); LV 2: one z-block per chunk; LV 0 (runtime
// level >= 3): the chunk lies inside one half (hh) of its z-block.
// The 8 fp64 multipliers of one Psi entry, computed ONCE per entry when its index
// batch is staged (k_split3c), not by every lane of the entry's group in every round:
//   LV > 0: {min(psi_t,0) t = A,H,V,D;  min(-psi_A,0);  TRICK ? psi_t : min(-psi_t,0) t = H,V,D}
//   LV 0  : {min(psi_t,0) t = A,H,V,D;  min(-psi_t,0) t = A,H,V,D}   (low-half / high-half sets)
// min/max in fp32 (FMNMX), then exact conversions; c^l is applied once per output.
template <int LV, bool TRICK>
__device__ __forceinline__ void split3_multipliers(const float4& ps, double (&m)[8]) {
    const float pf[4] = {ps.x, ps.y, ps.z, ps.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) m[t] = (double)fminf(pf[t], 0.f);
    m[4] = (double)fminf(-pf[0], 0.f);
#pragma unroll
    for (int t = 1; t < 4; ++t) m[4 + t] = (LV > 0 && TRICK) ? (double)pf[t] : (double)fminf(-pf[t], 0.f);
}
template <int S, int LV, bool TRICK>
__device__ __forceinline__ void split3_consume(const double (&m)[8], const float (&f)[S], bool hh,
                                               double (&acc)[(S / 4) * (LV == 1 ? 14 : 7)]) {
    constexpr int V = S / 4;
    if constexpr (LV > 0) {
        constexpr int HS = LV;            // half size in slices: 1 or 2
        constexpr int NZ = 2 / HS;        // z-blocks per chunk
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
            for (int z = 0; z < NZ; ++z) {
                const float* fz = f + 4 * v + 2 * HS * z;
                double qlo = f2d_wide<false>(fz[0]), qhi = f2d_wide<false>(fz[HS]);
                if constexpr (HS == 2) {
                    qlo += f2d_wide<false>(fz[1]);
                    qhi += f2d_wide<false>(fz[3]);
                }
                const double qall = qlo + qhi;
                double* a = acc + 7 * (v * NZ + z);
#pragma unroll
                for (int t = 0; t < 3; ++t) a[t] = fma(m[1 + t], qall, a[t]);
                a[3] = fma(m[4], qhi, fma(m[0], qlo, a[3]));
#pragma unroll
                for (int t = 0; t < 3; ++t) {
                    if constexpr (TRICK) a[4 + t] = fma(m[5 + t], qhi, a[4 + t]);
                    else a[4 + t] = fma(m[5 + t], qhi, fma(m[1 + t], qlo, a[4 + t]));
                }
            }
    } else {
        // z-low: min(psi_t,0), t = H,V,D; z-high: this lane's half (low: min(psi,0), high: min(-psi,0))
        double mh[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) mh[t] = hh ? m[4 + t] : m[t];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            double qs = f2d_wide<false>(f[4 * v]);
#pragma unroll
            for (int i = 1; i < 4; ++i) qs += f2d_wide<false>(f[4 * v + i]);
#pragma unroll
            for (int t = 0; t < 3; ++t) acc[7 * v + t] = fma(m[1 + t], qs, acc[7 * v + t]);
#pragma unroll
            for (int t = 0; t < 4; ++t) acc[7 * v + 3 + t] = fma(mh[t], qs, acc[7 * v + 3 + t]);
        }
    }
}
template <int P, int E, int D, int WPI>
struct Split3cSmem {
    static constexpr int S = P * E / 32;
    float4 ring[4][D][S / 4][32];   // [warp][round % D][16-byte part][lane]
    unsigned iray[4][2][32];        // [warp][batch % 2][entry]
    double2 imul[4][2][4][32];      // [warp][batch % 2][multiplier pair][entry]: 8 fp64 multipliers per entry
    double red[4][7][P / 2];
};
template <int P, int E, int LV, bool TRICK, int D, int WPI>
__device__ __forceinline__ void split3c_block(unsigned b, int l, int lane, int wib, int nx, int ny, int nzl,
                                              uint64_t e0, uint64_t e1, const unsigned* __restrict__ eray,
                                              const float4* __restrict__ epsi, const float* __restrict__ q,
                                              const uint8_t* __restrict__ act, const ActOff& off,
                                              double* __restrict__ bm, const TileMap& tmap,
                                              Split3cSmem<P, E, D, WPI>& sm) {
    constexpr int LPE = 32 / E, S = P * E / 32;
    static_assert(S == 4 || S == 8, "slices per lane");
    static_assert(32 % E == 0 && (32 / E) >= 1, "entry groups");
    static_assert(LV >= 0 && LV <= 2, "levels 1 and 2 are specialised; 0 = runtime level >= 3");
    constexpr int V = S / 4;                        // chunks of 4 consecutive slices per lane
    constexpr int NZC = LV == 1 ? 2 : 1;            // z-blocks (LV > 0) or partials (LV 0) per chunk
    constexpr int NA = V * (LV == 1 ? 14 : 7);
    constexpr int RPB = 32 / E;   // rounds per index batch (32 entries)
    static_assert(D >= 2 && D - 1 <= RPB, "the ring may reach at most one index batch ahead");
    const int grp = lane / LPE, j = lane % LPE;
    const bool hh = LV == 0 ? (((4 * j) >> (l - 1)) & 1) != 0 : false;   // 4*LPE*v is a multiple of 2^l
    double acc[NA];
#pragma unroll
    for (int i = 0; i < NA; ++i) acc[i] = 0.0;
    // this warp's entries [ws, we): contiguous chunks, multiples of 32 entries
    const int wi = WPI == 1 ? 0 : wib;
    const uint64_t n = e1 - e0;
    const uint64_t chunk = ((n + WPI - 1) / WPI + 31) / 32 * 32;
    const uint64_t ws0 = e0 + (uint64_t)wi * chunk, ws = ws0 < e1 ? ws0 : e1, we = ws + chunk < e1 ? ws + chunk : e1;
    const uint64_t nr = (we - ws + E - 1) / E;
    const uint64_t nbat = (we - ws + 31) / 32;
    unsigned ry = 0;
    float4 rp = make_float4(0.f, 0.f, 0.f, 0.f);
    auto ldg_batch = [&](uint64_t k) {   // lane i: entry ws + 32k + i
        const uint64_t ee = ws + 32 * k + lane;
        const bool ok = ee < we;
        ry = __ldg(eray + (ok ? ee : ws));
        rp = ok ? __ldg(epsi + ee) : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    auto sts_batch = [&](uint64_t k) {
        sm.iray[wib][k & 1][lane] = ry;
        double m[8];
        split3_multipliers<LV, TRICK>(rp, m);
#pragma unroll
        for (int t = 0; t < 4; ++t) sm.imul[wib][k & 1][t][lane] = make_double2(m[2 * t], m[2 * t + 1]);
    };
    auto issue_q = [&](uint64_t r) {   // q row parts of round r into ring slot r % D
        if (r < nr) {
            const unsigned y = sm.iray[wib][(r / RPB) & 1][(r % RPB) * E + grp];
            const float4* row = reinterpret_cast<const float4*>(q + (uint64_t)y * P) + j;
#pragma unroll
            for (int v = 0; v < S / 4; ++v) cp_async16(&sm.ring[wib][r % D][v][lane], row + LPE * v);
        }
        cp_async_commit();
    };
    if (nr > 0) {
        ldg_batch(0);
        sts_batch(0);
        if (nbat > 1) ldg_batch(1);
        __syncwarp();
#pragma unroll
        for (int r = 0; r < D - 1; ++r) issue_q(r);   // all in batch 0 (D - 1 <= RPB)
        for (uint64_t r = 0; r < nr; ++r) {
            const uint64_t ra = r + D - 1;   // round whose q goes out now
            if (ra % RPB == 0 && ra / RPB < nbat) {
                const uint64_t k = ra / RPB;   // batch k's registers -> shared, fetch batch k + 1
                __syncwarp();                  // every lane is done reading buffer k & 1 (batch k - 2)
                sts_batch(k);
                if (k + 1 < nbat) ldg_batch(k + 1);
                __syncwarp();
            }
            issue_q(ra);
            double m[8];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const double2 mm = sm.imul[wib][(r / RPB) & 1][t][(r % RPB) * E + grp];
                m[2 * t] = mm.x; m[2 * t + 1] = mm.y;
            }
            cp_async_wait<D - 1>();
            float f[S];
#pragma unroll
            for (int v = 0; v < S / 4; ++v) {
                const float4 t4 = sm.ring[wib][r % D][v][lane];
                f[4 * v] = t4.x; f[4 * v + 1] = t4.y; f[4 * v + 2] = t4.z; f[4 * v + 3] = t4.w;
            }
            split3_consume<S, LV, TRICK>(m, f, hh, acc);
        }
        cp_async_wait<0>();
    }
    if constexpr (LV > 0 && TRICK) {
#pragma unroll
        for (int z = 0; z < V * NZC; ++z)
#pragma unroll
            for (int t = 0; t < 3; ++t) acc[7 * z + 4 + t] = acc[7 * z + t] - acc[7 * z + 4 + t];
    }
#pragma unroll
    for (int o = LPE; o < 32; o <<= 1)
#pragma unroll
        for (int i = 0; i < NA; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
    // red slot = z-block index (LV > 0) or chunk index in slice order (LV 0: 4 slices per slot)
    if (grp == 0) {
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
            for (int z = 0; z < NZC; ++z)
#pragma unroll
                for (int t = 0; t < 7; ++t)
                    sm.red[wib][t][(LPE * v + j) * NZC + z] = acc[7 * (v * NZC + z) + t];
    }
    if constexpr (WPI == 1) __syncwarp(); else __syncthreads();
    const double cls = cpow3(l) * kTwo896;
    const int nk = nzl >> l, hl = ny >> l, wl = nx >> l, dl = nk;
    const int bi = (int)(b / wl), bj = (int)(b % wl);
    const int per = LV > 0 ? 1 : ((1 << l) / 4);   // red slots per z-block
    const int t0 = WPI == 1 ? lane : (int)threadIdx.x, tstep = WPI == 1 ? 32 : 32 * WPI;
    for (int k = t0; k < nk; k += tstep) {
        if (!act[off.off[l] + ((uint64_t)k * hl + bi) * wl + bj]) continue;
        const int zz[7] = {k, k, k, dl + k, dl + k, dl + k, dl + k};
        const int yy[7] = {hl + bi, bi, hl + bi, bi, hl + bi, bi, hl + bi};
        const int xx[7] = {bj, wl + bj, wl + bj, bj, bj, wl + bj, wl + bj};
#pragma unroll
        for (int t = 0; t < 7; ++t) {
            double tot = 0.0;
            for (int w = (WPI == 1 ? wib : 0); w < (WPI == 1 ? wib + 1 : WPI); ++w) {   // warp order
                double sum = sm.red[w][t][k * per];
                for (int gg = 1; gg < per; ++gg) sum += sm.red[w][t][k * per + gg];
                tot = (WPI == 1) ? sum : tot + sum;
            }
            bm[tmap.L ? coef_tile_pos(tmap, l, yy[t], xx[t], zz[t]) : ((uint64_t)yy[t] * nx + xx[t]) * P + zz[t]] =
                tot * cls;
        }
    }
    if constexpr (WPI == 1) __syncwarp(); else __syncthreads();
}
template <int P, int E, bool TRICK, int D, int WPI, int MINB>
__global__ void __launch_bounds__(128, MINB) k_split3c(uint64_t nlist, const uint2* __restrict__ list, int nx, int ny,
                                                       int nzl, const unsigned long long* __restrict__ ptr,
                                                       const unsigned* __restrict__ eray,
                                                       const float4* __restrict__ epsi, const float* __restrict__ q,
                                                       const uint8_t* __restrict__ act, ActOff off, ActOff koff,
                                                       double* __restrict__ bm, TileMap tmap,
                                                       unsigned long long* __restrict__ ctr) {
    static_assert(WPI == 1 || WPI == 4, "warps per item");
    constexpr int S = P * E / 32;
    __shared__ Split3cSmem<P, E, D, WPI> sm;
    __shared__ unsigned long long s_it;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    // Items are handed out in list (Morton) order from one counter, so the blocks
    // in flight are always consecutive list items: a static grid stride lets the
    // workers drift apart (items differ 2x in length) and with them the window of
    // q rows that should stay in L2.
    for (;;) {
        uint64_t it;
        if constexpr (WPI == 1) {
            unsigned long long v = 0;
            if (lane == 0) v = atomicAdd(ctr, 1ull);
            it = __shfl_sync(0xffffffffu, v, 0);
        } else {
            if (threadIdx.x == 0) s_it = atomicAdd(ctr, 1ull);
            __syncthreads();
            it = s_it;
            __syncthreads();
        }
        if (it >= nlist) break;
        const unsigned b = list[it].x;
        const int l = (int)list[it].y;
        const uint64_t key = koff.off[l] + b;
        const uint64_t e0 = ptr[key], e1 = ptr[key + 1];
#define SP(LVv) split3c_block<P, E, LVv, TRICK, D, WPI>(b, l, lane, wib, nx, ny, nzl, e0, e1, eray, epsi, q, act, off, bm, tmap, sm)
        if (l == 1) SP(1);
        else if (l == 2) SP(2);
        else SP(0);
#undef SP
    }
}

// ---- split, lane per ACTIVE z-block (opt-in WAMGPU_SPLIT_VARIANT=7; measured 2x
// slower than k_split3h_e: its 8-byte per-lane q loads are scattered over the row,
// the multipliers are prepared per z-block instead of per 4 z-blocks, and most
// z-blocks of a listed block turn out to be active).  k_split3h_e spends the same
// work on every z-block of a listed in-plane block, but at the BASELINE trees
// only ~1/3 of them are active (cfg4 final tree: 6.3e6 of 1.7e7 level-1 blocks),
// and it issues both products of every z-high coefficient although one of its
// two multipliers is always zero.  Here the warp compacts the block's active
// z-blocks from its z-bit words; lane j of an entry group owns the j-th active
// z-block (and the (j+32)-th when more than 32 are active) and follows the
// per-half formulation of the SPEC split (separable model): per entry
//   qlo / qhi = slice-order sums of q over the z-block's halves, qall = qlo + qhi,
//   z-low  p in H,V,D:   acc += (p < 0 ? p : 0) * qall
//   z-high p in A,H,V,D: acc += p < 0 ? p * qlo : -p * qhi        (p = psi c^l)
// i.e. 7 FMAs per (entry, active z-block).  32/lpe entry groups run side by
// side (lpe = lanes per entry = the active count rounded up to a power of two)
// and are combined by a fixed xor butterfly.  psi is moved into fp64 by the
// exact bit move (f2d_scaled, times cl * 2^896: bit-identical to (double)psi * cl).
template <int LL>
__device__ __forceinline__ void split3z_q(const float* __restrict__ qrow, int k, double& qlo, double& qhi) {
    constexpr int HW = 1 << (LL - 1);
    const float* p = qrow + ((size_t)k << LL);
    float f[2 * HW];
    if constexpr (LL == 1) {
        const float2 v = __ldg(reinterpret_cast<const float2*>(p));
        f[0] = v.x; f[1] = v.y;
    } else {
#pragma unroll
        for (int i = 0; i < HW / 2; ++i) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(p) + i);
            f[4 * i] = v.x; f[4 * i + 1] = v.y; f[4 * i + 2] = v.z; f[4 * i + 3] = v.w;
        }
    }
    qlo = 0.0; qhi = 0.0;
#pragma unroll
    for (int i = 0; i < HW; ++i) qlo += (double)f[i];
#pragma unroll
    for (int i = 0; i < HW; ++i) qhi += (double)f[HW + i];
}
__device__ __forceinline__ int nth_set64(unsigned w0, unsigned w1, int n) {   // n-th (0-based) set bit of w1:w0
    const int c0 = __popc(w0);
    return n < c0 ? (int)__fns(w0, 0, n + 1) : 32 + (int)__fns(w1, 0, n - c0 + 1);
}
template <int P, int LL>
__device__ __forceinline__ void split3z_block(unsigned b, int lane, unsigned w0, unsigned w1, int na, int nx, int ny,
                                              int nzl, uint64_t e0, uint64_t e1, const unsigned* __restrict__ eray,
                                              const float4* __restrict__ epsi, const float* __restrict__ q,
                                              double* __restrict__ bm, const TileMap& tmap) {
    const int lpe = na > 16 ? 32 : (na > 8 ? 16 : (na > 4 ? 8 : (na > 2 ? 4 : (na > 1 ? 2 : 1))));
    const int E = 32 / lpe, grp = lane / lpe, j = lane % lpe;
    const int k0 = j < na ? nth_set64(w0, w1, j) : -1;
    const int k1 = j + 32 < na ? nth_set64(w0, w1, j + 32) : -1;
    const bool two = na > 32;   // warp-uniform
    const double cls = cpow3(LL) * kTwo896;
    double acc[2][7];
#pragma unroll
    for (int z = 0; z < 2; ++z)
#pragma unroll
        for (int t = 0; t < 7; ++t) acc[z][t] = 0.0;
    auto step = [&](const float4& ps, double qlo, double qhi, double (&a)[7]) {
        const double qall = qlo + qhi;
        const float pf[4] = {ps.x, ps.y, ps.z, ps.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const double pc = f2d_scaled<true>(pf[t]) * cls;   // == (double)psi * c^l
            const bool neg = pf[t] < 0.0f;
            if (t > 0) a[t - 1] = fma(neg ? pc : 0.0, qall, a[t - 1]);
            a[3 + t] = fma(neg ? pc : -pc, neg ? qlo : qhi, a[3 + t]);
        }
    };
    // software pipeline: entry e + E's ray, psi and q values are in flight while e is consumed
    uint64_t e = e0 + grp;
    unsigned yn = 0;
    float4 pn = make_float4(0.f, 0.f, 0.f, 0.f);
    double l0 = 0.0, h0 = 0.0, l1 = 0.0, h1 = 0.0;
    auto fetch = [&](uint64_t ee) {
        if (ee < e1) {
            yn = __ldg(eray + ee);
            pn = __ldg(epsi + ee);
            const float* qrow = q + (uint64_t)yn * P;
            if (k0 >= 0) split3z_q<LL>(qrow, k0, l0, h0);
            if (two && k1 >= 0) split3z_q<LL>(qrow, k1, l1, h1);
        }
    };
    fetch(e);
    while (e < e1) {
        const float4 pc4 = pn;
        const double cl0 = l0, ch0 = h0, cl1 = l1, ch1 = h1;
        fetch(e + E);
        if (k0 >= 0) step(pc4, cl0, ch0, acc[0]);
        if (two && k1 >= 0) step(pc4, cl1, ch1, acc[1]);
        e += E;
    }
    // combine the entry groups (lanes j, j + lpe, ...): fixed order
    for (int o = lpe; o < 32; o <<= 1)
#pragma unroll
        for (int z = 0; z < 2; ++z)
#pragma unroll
            for (int t = 0; t < 7; ++t) acc[z][t] += __shfl_xor_sync(0xffffffffu, acc[z][t], o);
    if (grp == 0) {
        const int hl = ny >> LL, wl = nx >> LL, dl = nzl >> LL;
        const int bi = (int)(b / wl), bj = (int)(b % wl);
#pragma unroll
        for (int z = 0; z < 2; ++z) {
            const int k = z ? k1 : k0;
            if (k < 0) continue;
            const int zz[7] = {k, k, k, dl + k, dl + k, dl + k, dl + k};
            const int yy[7] = {hl + bi, bi, hl + bi, bi, hl + bi, bi, hl + bi};
            const int xx[7] = {bj, wl + bj, wl + bj, bj, bj, wl + bj, wl + bj};
#pragma unroll
            for (int t = 0; t < 7; ++t)
                bm[tmap.L ? coef_tile_pos(tmap, LL, yy[t], xx[t], zz[t]) : ((uint64_t)yy[t] * nx + xx[t]) * P + zz[t]] =
                    acc[z][t];
        }
    }
}
template <int P>
__global__ void __launch_bounds__(128) k_split3z(uint64_t nlist, const uint2* __restrict__ list, int nx, int ny,
                                                 int nzl, const unsigned long long* __restrict__ ptr,
                                                 const unsigned* __restrict__ eray, const float4* __restrict__ epsi,
                                                 const float* __restrict__ q, const unsigned* __restrict__ zbits,
                                                 ActOff zoff, ActOff koff, double* __restrict__ bm, TileMap tmap) {
    const int lane = threadIdx.x & 31;
    const uint64_t W = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t it = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < nlist; it += W) {
        const unsigned b = list[it].x;
        const int l = (int)list[it].y;
        const int nk = nzl >> l, nw = (nk + 31) >> 5;
        const unsigned* zb = zbits + zoff.off[l] + (uint64_t)b * nw;
        const unsigned w0 = zb[0], w1 = nw > 1 ? zb[1] : 0u;
        const int na = __popc(w0) + __popc(w1);
        if (na == 0) continue;
        const uint64_t key = koff.off[l] + b;
        const uint64_t e0 = ptr[key], e1 = ptr[key + 1];
#define SZ(LLv) case LLv: if constexpr ((P >> LLv) >= 1) split3z_block<P, LLv>(b, lane, w0, w1, na, nx, ny, nzl, e0, e1, eray, epsi, q, bm, tmap); break;
        switch (l) { SZ(1) SZ(2) SZ(3) SZ(4) SZ(5) default: break; }
#undef SZ
    }
}

// Ray bands of the 3D split.  The split gathers one P*4-byte row of q per Psi
// entry; a block's list holds every view, and the q slab outgrows L2 at the
// BASELINE sizes (cfg4: 755 MB, so the final tree's 8.7e8 entries re-read
// 444 GB from DRAM per split).  Cutting the rays into B bands whose q rows stay
// L2-resident and running the split band by band turns that into L2 hits.
// Lists are sorted by (key, ray), so a band is one contiguous range per key:
// bptr[key*(B+1) + b] = first entry of `key` with ray >= b*rpb (b = B: its end).
__global__ void k_split_band_ptr(uint64_t nkeys, const unsigned long long* __restrict__ ptr,
                                 const unsigned* __restrict__ eray, int B, unsigned rpb,
                                 unsigned long long* __restrict__ bptr) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nkeys * (uint64_t)(B + 1)) return;
    const uint64_t key = i / (B + 1);
    const int b = (int)(i % (B + 1));
    uint64_t lo = ptr[key], hi = ptr[key + 1];
    if (b == B) { bptr[i] = hi; return; }
    const unsigned r0 = (unsigned)b * rpb;
    while (lo < hi) {   // lower bound of r0
        const uint64_t mid = (lo + hi) >> 1;
        if (eray[mid] < r0) lo = mid + 1;
        else hi = mid;
    }
    bptr[i] = lo;
}

}  // namespace wamgpu
