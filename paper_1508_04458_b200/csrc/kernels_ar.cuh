// kernels_ar.cuh — fused back projection + all-reduce over NVLink peer memory
// (multi-GPU 2D view sharding).
//
// With views sharded, every rank holds a partial [g || b-] (g = H^T q over its
// own rays, b- the signed split over its own Phi- rows) and every rank needs
// the sum.  Instead of a back-projection kernel followed by ncclAllReduce, ONE
// persistent kernel per rank does both, tile by tile:
//   phase 1  each CTA computes a 256-element tile of its partial and stores it
//            straight into the tile OWNER's staging slot on the owner's GPU
//            (st.global to a peer-mapped pointer), then signals the owner with a
//            system-scope atomic on the owner's per-tile counter.  The NVLink
//            transfer of tile t overlaps the computation of tile t+1.
//   phase 2  the owner of a tile (tile % R) waits for its R contributions, sums
//            them in RANK ORDER (deterministic; identical on every rank) and
//            stores the result into every rank's result buffer (peer stores),
//            signalling each rank's ready counter.
//   phase 3  a rank returns once all tiles of its result have arrived.
// Counters are monotonic (epoch e waits for e*R arrivals / e*ntiles tiles), so
// nothing is reset between calls.  A rank only overwrites a peer's staging slot
// in epoch e+1 after it has received every tile of epoch e, i.e. after each
// owner has finished reading its slot: no overlap between epochs.
// All CTAs spin on one another, so the kernel is launched cooperatively (all
// CTAs resident).  The same kernel runs R LOGICAL ranks in one grid on one GPU
// (rexec = R, CTAs partitioned per logical rank): that is how the protocol is
// tested without R GPUs (B200_PROFILING.md: emulate the ranks as one kernel).
#pragma once
#include <cstdint>

namespace wamgpu {

constexpr int AR_MAX = 8;      // ranks per NVLink/NVSwitch node
constexpr int AR_TILE = 256;   // doubles per tile (2 KB)

struct ArArgs {
    double* slot[AR_MAX];              // rank k's staging area: R x n doubles (slot + src*n + i)
    double* res[AR_MAX];               // rank k's result vector: n doubles
    unsigned long long* cnt[AR_MAX];   // rank k's per-tile arrival counters: ntiles
    unsigned long long* rdy[AR_MAX];   // rank k's tiles-ready counter: 1
    uint64_t n;                        // vector length
    unsigned long long epoch;          // 1, 2, ... identical on every rank
    int R;                             // world size
    int r0, rexec;                     // logical ranks run by this launch: [r0, r0 + rexec)
    int* err;                          // bit 8 set when a wait exceeds AR_TIMEOUT_NS
};
constexpr unsigned long long AR_TIMEOUT_NS = 10ull * 1000 * 1000 * 1000;   // 10 s: a peer never arrived

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// spin until *p >= target; false (and err |= 256) after AR_TIMEOUT_NS
__device__ __forceinline__ bool ar_wait(const unsigned long long* p, unsigned long long target, int* err) {
    const unsigned long long t0 = globaltimer_ns();
    while (true) {
        unsigned long long v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
        if (v >= target) return true;
        if (globaltimer_ns() - t0 > AR_TIMEOUT_NS) {
            atomicOr(err, 256);
            return false;
        }
        __nanosleep(64);
    }
}

// Self-test / emulation producer: the partial of logical rank r is in[r][0..n).
struct ArProdCopy {
    const double* in[AR_MAX];
    __device__ __forceinline__ void tile(int me, uint64_t base, int len, double* sv) const {
        for (int i = threadIdx.x; i < len; i += blockDim.x) sv[i] = in[me][base + i];
        __syncthreads();
    }
};

// Production producer: [g || extra] with g(x) = sum_y h(y|x) w(y) over this
// rank's CSC columns (seg_dot<1,12>: bit-identical to k_back<0,12,1>) and
// extra = the rank's partial signed split (or zeros).
// (Per-rank tables: a launch that emulates R ranks gives each logical rank its
// own shard; a production launch fills only entry [rank].)
struct ArProdBack {
    const unsigned long long* cp[AR_MAX];
    const uint2* C[AR_MAX];
    const float* w[AR_MAX];
    const double* extra[AR_MAX];
    uint64_t N;
    __device__ __forceinline__ void tile(int me, uint64_t base, int len, double* sv) const {
        const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (int i = wib; i < len; i += nw) {
            const uint64_t x = base + i;
            if (x < N) {
                const uint64_t nob[1] = {0};
                double cc[1];
                seg_dot<1, 12>(C[me], w[me], cp[me][x], nob, cp[me][x + 1], lane, cc);
                if (lane == 0) sv[i] = cc[0];
            } else if (lane == 0) {
                sv[i] = extra[me][x - N];
            }
        }
        __syncthreads();
    }
};

template <class Prod>
__global__ void __launch_bounds__(256) k_fused_allreduce(ArArgs a, Prod prod) {
    __shared__ double sv[AR_TILE];
    const uint64_t ntiles = (a.n + AR_TILE - 1) / AR_TILE;
    const int per = (int)gridDim.x / a.rexec;   // CTAs per executed logical rank
    const int me = a.r0 + (int)blockIdx.x / per, cta = (int)blockIdx.x % per;
    // phase 1: produce every tile of my partial, push it to the tile's owner
    for (uint64_t t = cta; t < ntiles; t += per) {
        const uint64_t base = t * AR_TILE;
        const int len = (int)min((uint64_t)AR_TILE, a.n - base);
        prod.tile(me, base, len, sv);
        const int owner = (int)(t % (uint64_t)a.R);
        double* dst = a.slot[owner] + (uint64_t)me * a.n + base;
        for (int i = threadIdx.x; i < len; i += blockDim.x) dst[i] = sv[i];
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) atomicAdd_system(a.cnt[owner] + t, 1ull);
        __syncthreads();   // sv is reused by the next tile
    }
    // phase 2: reduce the tiles I own (t % R == me), in rank order, broadcast
    for (uint64_t t = (uint64_t)me + (uint64_t)a.R * cta; t < ntiles; t += (uint64_t)a.R * per) {
        __shared__ int s_ok;
        if (threadIdx.x == 0) s_ok = ar_wait(a.cnt[me] + t, a.epoch * (unsigned long long)a.R, a.err);
        __syncthreads();
        if (!s_ok) return;   // a peer never arrived: err is set, the host raises
        const uint64_t base = t * AR_TILE;
        const int len = (int)min((uint64_t)AR_TILE, a.n - base);
        for (int i = threadIdx.x; i < len; i += blockDim.x) {
            double s = 0.0;
            for (int k = 0; k < a.R; ++k) s += __ldcg(a.slot[me] + (uint64_t)k * a.n + base + i);
            for (int j = 0; j < a.R; ++j) a.res[j][base + i] = s;
        }
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0)
            for (int j = 0; j < a.R; ++j) atomicAdd_system(a.rdy[j], 1ull);
    }
    // phase 3: my result is complete once every tile has been broadcast to me
    if (cta == 0 && threadIdx.x == 0) ar_wait(a.rdy[me], a.epoch * (unsigned long long)ntiles, a.err);
    __syncthreads();
}

}  // namespace wamgpu
