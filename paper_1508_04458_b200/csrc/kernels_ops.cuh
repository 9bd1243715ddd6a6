// Standalone core-model ops of SPEC.md:81-98 (predicted_means, i_divergence) on
// vectors the caller supplies.  The iteration never calls these: its forward
// kernels fuse Beer's law and the I-divergence partials (k_fwd_patch, k_fwd3s).
// Both are pure streams (24 B and 16 B per ray), grid-stride over a grid of a
// multiple of the SM count; sums are fixed-order (per-thread stride, xor
// butterfly, per-warp slots, then k_sum_partials), so a call is reproducible.
#pragma once
#include <cstdint>

namespace wamgpu {

// q(y) = I0(y) exp(-l(y)).  bad[0] = smallest ray index with a non-finite l
// ("numerical error with ray index"), ~0 when none.
__global__ void __launch_bounds__(256)
k_pred_means(const double* __restrict__ I0, const double* __restrict__ l, double* __restrict__ q, uint64_t n,
             unsigned long long* __restrict__ bad) {
    unsigned long long first = ~0ull;
    for (uint64_t y = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; y < n; y += (uint64_t)gridDim.x * blockDim.x) {
        const double ly = l[y];
        if (!isfinite(ly)) { if (y < first) first = y; continue; }
        q[y] = I0[y] * exp(-ly);
    }
    if (first != ~0ull) atomicMin(bad, first);
}

// part[block] = sum over the block's rays of d log(d/q) - d + q (0 log 0 = 0,
// SPEC.md:92); bad[0] = smallest ray index with q <= 0 (or NaN).
__global__ void __launch_bounds__(256)
k_idiv_partials(const double* __restrict__ d, const double* __restrict__ q, uint64_t n, double* __restrict__ part,
                unsigned long long* __restrict__ bad) {
    unsigned long long first = ~0ull;
    double a = 0.0;
    for (uint64_t y = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; y < n; y += (uint64_t)gridDim.x * blockDim.x) {
        const double dy = d[y], qy = q[y];
        if (!(qy > 0.0)) { if (y < first) first = y; continue; }
        a += (dy > 0.0 ? dy * log(dy / qy) : 0.0) - dy + qy;
    }
    a = warp_sum(a);
    __shared__ double s[8];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        double r = 0.0;
        for (int w = 0; w < 8; ++w) r += s[w];
        part[blockIdx.x] = r;
    }
    if (first != ~0ull) atomicMin(bad, first);
}

}  // namespace wamgpu
