// wamgpu.cu — host orchestration and C-ABI of libwamgpu.so (include/wamgpu.h).
//
// One context per GPU.  Per wavelet-AM iteration (PAPER.md
// Algorithm 1) the context launches, on its own stream:
//   k_back<0>   g = H^T q                      (CSC gather, fp64)      K3
//   k_split     b-(z) over Phi^- columns        (active details only)  K5
//   [ncclAllReduce SUM fp64 over (g | b-)]      (view-sharded 2D only)
//   k_tile<1>   S = Omega^T g; b+ = S - b-; root solve; mu = Omega beta  K4+K6+K1
//   k_forward<1> l = H mu, q = I0 e^-l, I-div partials                  K2
//   k_sum_partials + [allreduce] + k_record
// At scheduled expansions: k_tile<0> (fp64 image) -> max -> k_mark ->
// k_walk<0> (Z0) -> k_walk<1,2> + counting placement (Phi^- CSC rebuild; radix
// sort under WAMGPU_PHI_SORT=1)                                         K7, K8.
// The AM baseline is k_back<1> (fused update) + k_forward<1>.
#include <cub/cub.cuh>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/wamgpu.h"
#include "host_model.hpp"
#include "kernels.cuh"
#include "kernels3d.cuh"
#include "kernels3h.cuh"
#include "kernels3t.cuh"
#include "kernels_ar.cuh"
#include "kernels_phi.cuh"
#include "kernels3c.cuh"
#include "kernels_ops.cuh"

namespace wamgpu {

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)
#define NK(x)                                                                                     \
    do {                                                                                          \
        ncclResult_t r_ = (x);                                                                    \
        if (r_ != ncclSuccess) throw CudaError(std::string(#x) + ": " + ncclGetErrorString(r_)); \
    } while (0)

// ---- guard bands (WAMGPU_GUARD=1, debug).  compute-sanitizer is closed on the
// GPU pool this was developed on (profiles/r06/sanitizer_memcheck_closed.log),
// so the library carries its own write-overrun and uninitialised-read check:
// every device allocation gets a 256-byte band of 0xA5 on both sides and its
// body is filled with 0xFF (NaN as fp32/fp64: a value read before it is written
// poisons the results and trips the NumericError flags / parity tests);
// wamgpu_debug_guards() verifies every live allocation's bands.
constexpr size_t kGuard = 256;
struct GuardReg {
    std::mutex m;
    std::map<void*, size_t> live;   // user pointer -> user bytes
};
static GuardReg& guard_reg() { static GuardReg g; return g; }
static bool guard_on() {
    static const bool on = [] { const char* e = std::getenv("WAMGPU_GUARD"); return e && std::atoi(e) != 0; }();
    return on;
}
static void* dev_malloc(size_t bytes) {
    void* p = nullptr;
    if (!guard_on()) { CK(cudaMalloc(&p, bytes)); return p; }
    char* raw = nullptr;
    CK(cudaMalloc(&raw, bytes + 2 * kGuard));
    CK(cudaMemset(raw, 0xA5, kGuard));
    CK(cudaMemset(raw + kGuard, 0xFF, bytes));
    CK(cudaMemset(raw + kGuard + bytes, 0xA5, kGuard));
    // the fills run on the default stream, asynchronously to the host and
    // unordered against the contexts' non-blocking streams: finish them before
    // anyone writes real data into the body
    CK(cudaStreamSynchronize(nullptr));
    p = raw + kGuard;
    std::lock_guard<std::mutex> l(guard_reg().m);
    guard_reg().live[p] = bytes;
    return p;
}
static void dev_free(void* p) {
    if (!guard_on()) { cudaFree(p); return; }
    {
        std::lock_guard<std::mutex> l(guard_reg().m);
        guard_reg().live.erase(p);
    }
    cudaFree(static_cast<char*>(p) - kGuard);
}
// (checked, bad): every live allocation's two bands compared with 0xA5
static std::pair<uint64_t, uint64_t> check_guards(std::string* first_bad) {
    uint64_t n = 0, bad = 0;
    if (!guard_on()) return {0, 0};
    CK(cudaDeviceSynchronize());
    std::lock_guard<std::mutex> l(guard_reg().m);
    std::vector<unsigned char> h(2 * kGuard);
    for (auto& kv : guard_reg().live) {
        char* u = static_cast<char*>(kv.first);
        CK(cudaMemcpy(h.data(), u - kGuard, kGuard, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(h.data() + kGuard, u + kv.second, kGuard, cudaMemcpyDeviceToHost));
        ++n;
        for (size_t i = 0; i < 2 * kGuard; ++i)
            if (h[i] != 0xA5) {
                ++bad;
                if (first_bad && first_bad->empty())
                    *first_bad = "allocation of " + std::to_string(kv.second) + " bytes: " +
                                 (i < kGuard ? "byte " + std::to_string((long)i - (long)kGuard) + " before its start"
                                             : "byte " + std::to_string(i - kGuard) + " past its end") + " overwritten";
                break;
            }
    }
    return {n, bad};
}

template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void alloc(size_t n_) {
        release();
        if (n_) p = static_cast<T*>(dev_malloc(n_ * sizeof(T)));
        n = n_;
    }
    void ensure(size_t n_) { if (n < n_) alloc(n_); }
    // streamed arrays get a 64-element tail so predicated vector/prefetch
    // loads just past the logical end stay inside the allocation
    void alloc_padded(size_t n_) { alloc(n_ + 64); n = n_ + 64; }
    void ensure_padded(size_t n_) { if (n < n_ + 64) alloc_padded(n_); }
    void release() { if (p) dev_free(p); p = nullptr; n = 0; }
    void swap(DBuf& o) { std::swap(p, o.p); std::swap(n, o.n); }
};

enum Cat { T_FWD = 0, T_BACK, T_SPLIT, T_UPDATE, T_EXPAND, T_COMM, T_PHI, T_FWDC, T_BACKC, T_NCAT };

// In-process rank group (wamgpu_set_comm_local): R contexts driven by R host
// threads of one process.  Collectives are a device-side rank-order reduction
// over the members' staging buffers between two host barriers.
struct LocalGroup {
    std::mutex m;
    std::condition_variable cv;
    int n = 0, joined = 0, arrived = 0;
    uint64_t gen = 0;
    bool broken = false;
    std::vector<double*> stage;   // per-rank device staging
    std::vector<int> dev;
};

}  // namespace wamgpu

using wamgpu::DBuf;
using wamgpu::ActOff;
using wamgpu::Cat;
using wamgpu::T_NCAT;
using wamgpu::CudaError;

struct wamgpu_ctx {
    int device = 0;
    cudaStream_t st = nullptr;
    int sms = 148;
    std::string err;
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1;
    // rank grid (partition): Rv view groups x Rz z-slab groups, rank = zg*Rv + vg.
    // comm_v: ranks sharing my slab (partial back projections are summed over
    // it); comm_z: ranks sharing my views (z-summed criterion).  nullptr = the
    // global comm (or no exchange when that group has one rank).
    int vgroups_req = 0, Rv = 1, Rz = 1, vg = 0, zg = 0;
    ncclComm_t comm_v = nullptr, comm_z = nullptr;
    int comm_kind = 0;                  // 0 none, 1 NCCL, 2 in-process group, 3 detached shard
    std::shared_ptr<wamgpu::LocalGroup> lg;
    DBuf<double> gstage;                // in-process group staging
    DBuf<double> rs_send, rs_recv;      // view-group update: reduce-scatter buffers (tile-major)
    DBuf<float> ag_send, ag_recv;       // view-group update: all-gather buffers {mu plane, counts}
    DBuf<float> bown, ball;             // view-group update: own beta plane, gathered planes
    bool beta_dirty = false;            // slab-Mallat beta behind the gathered beta planes
    uint8_t* act_pin = nullptr;         // pinned host copy of the tree bytes (expansions)
    // Φ_A (kernels_phi.cuh): approximation columns of the 2D tree, CSR + CSC,
    // built once per (matrix, L); used while no detail coefficient is active
    bool phiA_ok = false, mu_stale = false, phiA_beta_ok = true, bown_stale = false;
    DBuf<float> phiA_mblk;              // 3D: fp32 synthesis of each root (forward multiplier)
    int phiA_L = -1;
    uint64_t phiA_nnz = 0;
    DBuf<unsigned long long> phiA_rp, phiA_cp;
    DBuf<unsigned> phiA_col, phiA_row;
    DBuf<double> phiA_val, phiA_valC, phiA_part;
    uint64_t act_pin_n = 0;
    cudaStream_t st2 = nullptr;         // side stream (overlapped reduce-scatter)
    cudaEvent_t ev_x = nullptr, ev_y = nullptr;
    std::vector<int> peers_on;          // devices peer access was enabled to
    const uint8_t* add_tree = nullptr;  // wamgpu_wam_expand_with: caller blocks (host, act_bytes)
    // grid / matrix
    int nx = 0, ny = 0, nz = 1;
    bool have_grid = false, have_matrix = false;
    uint64_t M = 0, N = 0, row0 = 0, row1 = 0, Ml = 0, nnz = 0;
    int s0 = 0, nzl = 1;                // local z-slab [s0, s0+nzl) of an axial 3D stack (nz > 1)
    DBuf<unsigned> order;               // 3D back projection: voxels in 16x16 tile order
    DBuf<unsigned long long> rp, cp;
    DBuf<uint2> A, C;
    // compressed CSR for the 2D forward (C2, kernels.cuh): per-row header, 2-bit
    // step codes, fp32 h; c2_ok = built and verified
    DBuf<uint2> c2_rh;
    DBuf<unsigned short> c2_codes;
    DBuf<float> c2_h;
    bool c2_ok = false;
    // data
    DBuf<float> d, I0, q;
    bool have_data = false;
    // state
    int algo = 0;  // 1 AM, 2 WAM
    DBuf<float> mu, beta, fscratch;
    DBuf<char> xfer;                        // device side of the boundary transposes
    void* pin[2] = {nullptr, nullptr};      // pinned host staging, double-buffered
    cudaEvent_t pin_ev[2] = {nullptr, nullptr};
    DBuf<double> g, bdata, bam, mu64, bp_dbg, bm_dbg, zrow, dscratch;
    DBuf<unsigned long long> wcnt;      // separable 3D: per-(ray, level) Psi counts of the walk
    DBuf<unsigned long long> cursor;    // Phi^- emission cursor of the expansion walk
    DBuf<long long> zfix, zfix2;        // 2D tree: per-ray Z(y) in 2^-32 fixed point (pin P8)
    DBuf<ulonglong2> cols;              // 2D tree: Phi^- range [lo, hi) of column z inside E
    DBuf<unsigned long long> ptmp;      // column bounds of one placed batch
    DBuf<unsigned long long> pcur;      // placement cursors (copy of ptmp)
    std::vector<uint8_t> act_phi;       // tree that Phi^- / zfix currently cover
    DBuf<double> zA;                    // per-ray approximation part of Z (tree-independent)
    int zA_L = -1;                      // zA cache key: (levels, haar3, rows) of the last init walk
    bool zA_h3 = false;
    uint64_t zA_r0 = 0, zA_Ml = 0;
    DBuf<uint8_t> cub_tmp;
    DBuf<unsigned> kin_s, kout_s;
    DBuf<uint2> vin_s;
    int L = 0;
    DBuf<uint8_t> act, act_new;
    DBuf<unsigned> tbits;               // bit-packed tree for the expansion walk
    ActOff boff{};                      // bit offset of level l in tbits
    int tree_words = 0;
    // separable 3D Haar model (pin P3)
    bool haar3 = false;
    DBuf<unsigned> zbits;               // per (level, in-plane block): z-block activity words
    ActOff zoff{}, koff{};              // word offset of level l in zbits; key offset of level l
    uint64_t nkeys3 = 0;
    DBuf<unsigned> E3ray, pray_s;
    DBuf<uint2> sidx3;                  // Psi sort output (persistent)
    DBuf<float4> E3psi, ppsi_s;
    DBuf<uint2> list3;                  // (in-plane block, level) with any active z-block
    // block-coarsened matrices Hc, c = 2^k (kernels3c.cuh): built once per matrix and level
    struct Coarse {
        bool ok = false;
        uint64_t nnz = 0, Nc = 0;
        DBuf<unsigned long long> rp, cp;
        DBuf<unsigned> col, row, order;
        DBuf<double> val, valC;
        int seg = 1;                          // column segments of the z-coarse back projection
        DBuf<unsigned long long> cpseg;       // seg > 1: Nc*seg + 1 segment bounds (k_seg_bounds)
    } coarse[6];   // index k = 1 .. LMAX
    DBuf<float> mu_c;                   // mu on the coarse grid (forward operand)
    DBuf<double> g_c;                   // block sums of g (coarse back projection)
    DBuf<double> l_c;                   // z-coarse line integrals [ray][z-group]
    DBuf<float> w_z;                    // z-group sums of q as hi/lo pairs
    int fine_level = 0;                 // finest level with an active block (0: none)
    int mu_c_k = -1;                    // mu_c holds the z-coarse mu of this k (written by the coarse-domain update)
    int stats_k = -1;                   // >= 0: bp_dbg / bm_dbg lack the levels <= k (coarse-domain update): refresh on read
    std::vector<std::vector<unsigned>> morton;   // per level: in-plane blocks in Morton order (host, cached)
    int morton_nx = 0, morton_ny = 0;
    uint64_t nlist3 = 0;
    int walk_nlev = 1;
    ActOff off{};
    uint64_t act_bytes = 0;
    std::vector<uint8_t> act_host;
    DBuf<unsigned long long> np;
    DBuf<uint2> E;
    DBuf<unsigned> list;
    uint64_t nlist = 0, nnz_phi = 0, phi_batch = 0;
    double Z0 = 0.0;
    DBuf<double> scal, partial;
    int nblk_row = 1, nblk_col = 1;
    int lgx = -1;   // 2D mu in 8x4 tiles (mu_addr) when >= 0
    int fwd_variant = 0, back_variant = 0;  // SpMV tuning knobs (WAMGPU_FWD_VARIANT / WAMGPU_BACK_VARIANT)
    int split_variant = 0;                  // WAMGPU_SPLIT_VARIANT
    int walk_variant = 0;                   // WAMGPU_WALK_VARIANT
    int slab_variant = 112;                 // WAMGPU_SLAB_VARIANT (3D slab SpMM)
    // banded 3D forward (kernels3d.cuh k_fwd3s_band): image rows cut into
    // band_B bands of band_hb rows; per (local ray, band) entry range
    int band_B = 0, band_hb = 0, band_P = 0;
    DBuf<unsigned> blo, bhi;
    DBuf<double> lacc;                      // running per-(ray, slice) sums between band launches
    // ray bands of the separable-3D split (kernels3h.cuh k_split_band_ptr)
    DBuf<unsigned long long> bptr3;
    int sband_B = 1;
    bool mu_nonneg = false;                 // AM: mu has no sign bit set (see am_init)
    // on-the-fly 3D forward with TMA-staged image tiles (kernels3t.cuh): the
    // local ray table stays on the device; fwd3t: 0 off, 1 on (first launch
    // checks the bundle geometry), 2 verified, -1 rejected (slab SpMM kept)
    DBuf<wamgpu::RayDev> rays_dev;
    int geo_V = 0, geo_D = 0;
    double geo_h = 0.0;
    int fwd3t = 0, fwd3t_req = 0, t3_cb = 64;
    DBuf<int> t3flag;
    const void* t3_ptr = nullptr;           // tensor maps are encoded per (pointer, stride)
    int t3_P = 0;
    CUtensorMap t3_mx{}, t3_my{};
    double t_trace = 0.0;                   // WAMGPU_TRACE_HOST phase clock
    // fused back projection + all-reduce over NVLink peer memory (kernels_ar.cuh)
    struct {
        bool on = false;                    // set by wamgpu_p2p_import after its self-check
        DBuf<double> slot, res, extra, ones;
        DBuf<unsigned long long> cnt, rdy;
        wamgpu::ArArgs args{};
        std::vector<void*> opened;          // peer pointers from cudaIpcOpenMemHandle
        uint64_t n = 0;
    } ar;
    DBuf<unsigned long long> counters;
    DBuf<int> flag, flag2, it;
    DBuf<unsigned long long> split_ctr;   // work counter of k_split3c
    DBuf<double> objs;
    DBuf<unsigned long long> cums;
    int iter = 0;
    int64_t active = 0;
    cudaEvent_t ev_t0 = nullptr, ev_a = nullptr, ev_b = nullptr;
    std::vector<cudaEvent_t> ev_iter;
    // timing
    bool ktime = false;
    wamgpu_timing tm{};
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tev[T_NCAT];
    size_t tev_used[T_NCAT] = {};
    int64_t launches = 0;

    void timer_begin(Cat c, cudaStream_t s = nullptr) {
        if (!ktime) return;
        auto& v = tev[c];
        if (tev_used[c] == v.size()) {
            cudaEvent_t a, b;
            CK(cudaEventCreate(&a));
            CK(cudaEventCreate(&b));
            v.push_back({a, b});
        }
        CK(cudaEventRecord(v[tev_used[c]].first, s ? s : st));
    }
    void timer_end(Cat c, cudaStream_t s = nullptr) {
        if (!ktime) return;
        CK(cudaEventRecord(tev[c][tev_used[c]].second, s ? s : st));
        tev_used[c]++;
    }
};

namespace wamgpu {
using Ctx = ::wamgpu_ctx;

static double host_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
static bool trace_host() {
    static const bool on = std::getenv("WAMGPU_TRACE_HOST") != nullptr;
    return on;
}
#define HTRACE(label)                                                                  \
    do {                                                                               \
        if (trace_host()) {                                                            \
            CK(cudaStreamSynchronize(c->st));                                          \
            const double t_ = host_ms();                                               \
            std::fprintf(stderr, "[wamgpu] %-28s %8.3f ms\n", label, t_ - c->t_trace); \
            c->t_trace = t_;                                                           \
        }                                                                              \
    } while (0)

static thread_local std::string g_err;
static std::mutex g_groups_m;
static std::map<int, std::shared_ptr<LocalGroup>> g_groups;   // in-process rank groups by key

// ------------------------------------------------------------- utilities
static double cpow3_host(int l) {  // c^l, same sequence of multiplications as the device / oracle
    double c = 1.0;
    for (int i = 0; i < l; ++i) c *= 0.70710678118654752440;
    return c;
}
static inline unsigned blocks_for(uint64_t n, unsigned bs) { return (unsigned)((n + bs - 1) / bs); }

static void launched(Ctx* c, int n = 1) { c->launches += n; }

static bool g_sync_check = std::getenv("WAMGPU_SYNC_CHECK") != nullptr;  // debug: sync + check every launch
static void check_launch(Ctx* c, const char* what = "kernel") {
    CK(cudaGetLastError());
    if (g_sync_check) {
        const cudaError_t e = cudaStreamSynchronize(c->st);
        if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
    }
    launched(c);
}

static void exclusive_scan_u64(Ctx* c, unsigned long long* inout, uint64_t n) {
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, inout, inout, (int64_t)n, c->st));
    c->cub_tmp.ensure(tb + 1);
    CK(cub::DeviceScan::ExclusiveSum(c->cub_tmp.p, tb, inout, inout, (int64_t)n, c->st));
    launched(c);
}

static int bits_for(uint64_t n) {
    int b = 1;
    while ((1ull << b) <= n) ++b;
    return b;
}

// stable sort of (key, value) pairs by key; output in keys_out / vals_out
static void sort_pairs(Ctx* c, DBuf<unsigned>& kin, DBuf<uint2>& vin, DBuf<unsigned>& kout, DBuf<uint2>& vout,
                       uint64_t n, uint64_t maxkey) {
    kout.ensure_padded(std::max<uint64_t>(n, 1));
    vout.ensure_padded(std::max<uint64_t>(n, 1));
    if (n == 0) return;
    const int bits = bits_for(maxkey);
    auto vi = reinterpret_cast<unsigned long long*>(vin.p);
    auto vo = reinterpret_cast<unsigned long long*>(vout.p);
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, kin.p, kout.p, vi, vo, (int64_t)n, 0, bits, c->st));
    c->cub_tmp.ensure(tb + 1);
    CK(cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tb, kin.p, kout.p, vi, vo, (int64_t)n, 0, bits, c->st));
    launched(c, 4);
}

// ---- collectives ------------------------------------------------------------
// Scope of a reduction in the rank grid (partition()):
//   ALL    every rank (objective, Z0, criterion max);
//   VIEWS  the ranks holding the same z-slab and different views: the partial
//          back projections [g || b-] of view shards are summed over it;
//   SLABS  the ranks holding the same views and different z-slabs: the
//          z-summed criterion image of the per-slice Haar model.
enum Scope { S_ALL = 0, S_VIEWS, S_SLABS };

static int scope_size(const Ctx* c, Scope s) {
    return s == S_ALL ? c->nranks : (s == S_VIEWS ? c->Rv : c->Rz);
}
static std::vector<int> scope_members(const Ctx* c, Scope s) {
    std::vector<int> m;
    if (s == S_ALL) for (int r = 0; r < c->nranks; ++r) m.push_back(r);
    else if (s == S_VIEWS) for (int v = 0; v < c->Rv; ++v) m.push_back(c->zg * c->Rv + v);
    else for (int z = 0; z < c->Rz; ++z) m.push_back(z * c->Rv + c->vg);
    return m;
}

static void group_barrier(LocalGroup& g) {
    std::unique_lock<std::mutex> lk(g.m);
    if (g.broken) throw CudaError("local group: broken by an earlier failure of a peer rank");
    const uint64_t my = g.gen;
    if (++g.arrived == g.n) {
        g.arrived = 0;
        ++g.gen;
        g.cv.notify_all();
        return;
    }
    const bool ok = g.cv.wait_for(lk, std::chrono::seconds(120), [&] { return g.gen != my || g.broken; });
    if (!ok || g.broken) {
        g.broken = true;
        g.cv.notify_all();
        throw CudaError("local group: a peer rank did not arrive within 120 s");
    }
}

// the reduction kernels read the members' staging directly: peer access to
// every other device of the group
static void ensure_peer(Ctx* c, int d) {
    if (d == c->device || std::find(c->peers_on.begin(), c->peers_on.end(), d) != c->peers_on.end()) return;
    const cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        throw CudaError(std::string("local group: no peer access: ") + cudaGetErrorString(e));
    cudaGetLastError();
    c->peers_on.push_back(d);
}

// in-process group: copy to my staging, barrier, rank-order reduction of the
// members' staging into buf (identical on every member), barrier
static void local_allreduce(Ctx* c, double* buf, size_t n, int op, const std::vector<int>& mem) {
    LocalGroup& g = *c->lg;
    if ((int)mem.size() > GROUP_MAX) throw ConfigError("local group: at most 16 ranks per reduction");
    if (c->gstage.n < n) c->gstage.alloc(n);
    {
        std::lock_guard<std::mutex> lk(g.m);
        g.stage[c->rank] = c->gstage.p;
    }
    CK(cudaMemcpyAsync(c->gstage.p, buf, n * 8, cudaMemcpyDeviceToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));
    group_barrier(g);
    GroupPtrs gp{};
    {
        std::lock_guard<std::mutex> lk(g.m);
        for (size_t j = 0; j < mem.size(); ++j) {
            gp.p[j] = g.stage[mem[j]];
            ensure_peer(c, g.dev[mem[j]]);
        }
    }
    k_group_reduce<<<std::max<unsigned>(1, std::min<unsigned>(blocks_for(n, 256), c->sms * 8)), 256, 0, c->st>>>(
        buf, gp, (int)mem.size(), n, op);
    check_launch(c, "k_group_reduce");
    CK(cudaStreamSynchronize(c->st));
    group_barrier(g);
}

static void allreduce(Ctx* c, double* buf, size_t n, int op, Scope s) {
    if (c->comm_kind == 0 || c->comm_kind == 3) return;   // single rank / detached shard
    if (c->comm_kind == 1) {
        ncclComm_t cm = s == S_ALL ? c->comm : (s == S_VIEWS ? c->comm_v : c->comm_z);
        if (!cm) {
            if (scope_size(c, s) == 1 && c->nranks > 1) return;   // a one-rank group: nothing to exchange
            cm = c->comm;                                          // the group is the whole communicator
        }
        c->timer_begin(T_COMM);
        NK(ncclAllReduce(buf, buf, n, ncclDouble, op ? ncclMax : ncclSum, cm, c->st));
        c->timer_end(T_COMM);
        return;
    }
    // in-process group: every rank calls every collective; one-rank scopes are
    // skipped identically on all of them
    if (scope_size(c, s) == 1) return;
    c->timer_begin(T_COMM);
    local_allreduce(c, buf, n, op, scope_members(c, s));
    c->timer_end(T_COMM);
}
// my index in the members of scope s (rank order)
static int scope_index(const Ctx* c, Scope s) { return s == S_ALL ? c->rank : (s == S_VIEWS ? c->vg : c->zg); }

static ncclComm_t scope_comm(const Ctx* c, Scope s) {
    ncclComm_t cm = s == S_ALL ? c->comm : (s == S_VIEWS ? c->comm_v : c->comm_z);
    return cm ? cm : c->comm;   // nullptr: the group is the whole communicator (or has one rank)
}

// recv (chunk doubles) = rank-order sum over the scope's members of their
// send[idx*chunk, (idx+1)*chunk) -- idx = my index in the scope
static void reduce_scatter(Ctx* c, const double* send, double* recv, size_t chunk, Scope s, cudaStream_t st = nullptr) {
    if (!st) st = c->st;
    const bool timed = st == c->st;   // device timers live on the main stream
    const int n = scope_size(c, s);
    if (n == 1 || c->comm_kind == 0 || c->comm_kind == 3) {
        CK(cudaMemcpyAsync(recv, send + (size_t)scope_index(c, s) * chunk, chunk * 8, cudaMemcpyDeviceToDevice, st));
        return;
    }
    if (timed) c->timer_begin(T_COMM);
    if (c->comm_kind == 1) {
        NK(ncclReduceScatter(send, recv, chunk, ncclDouble, ncclSum, scope_comm(c, s), st));
    } else {
        LocalGroup& g = *c->lg;
        const std::vector<int> mem = scope_members(c, s);
        if ((int)mem.size() > GROUP_MAX) throw ConfigError("local group: at most 16 ranks per reduction");
        const size_t tot = chunk * mem.size();
        if (c->gstage.n < tot) c->gstage.alloc(tot);
        { std::lock_guard<std::mutex> lk(g.m); g.stage[c->rank] = c->gstage.p; }
        CK(cudaMemcpyAsync(c->gstage.p, send, tot * 8, cudaMemcpyDeviceToDevice, st));
        CK(cudaStreamSynchronize(st));
        group_barrier(g);
        GroupPtrs gp{};
        {
            std::lock_guard<std::mutex> lk(g.m);
            for (size_t j = 0; j < mem.size(); ++j) {
                gp.p[j] = g.stage[mem[j]] + (size_t)scope_index(c, s) * chunk;
                ensure_peer(c, g.dev[mem[j]]);
            }
        }
        k_group_reduce<<<std::max<unsigned>(1, std::min<unsigned>(blocks_for(chunk, 256), c->sms * 8)), 256, 0,
                         st>>>(recv, gp, (int)mem.size(), chunk, 0);
        check_launch(c, "k_group_reduce");
        CK(cudaStreamSynchronize(st));
        group_barrier(g);
    }
    if (timed) c->timer_end(T_COMM);
}

// recv (n x bytes) = the members' send (bytes each) in rank order
static void all_gather(Ctx* c, const void* send, void* recv, size_t bytes, Scope s) {
    const int n = scope_size(c, s);
    char* rb = static_cast<char*>(recv);
    if (n == 1 || c->comm_kind == 0) {
        if (rb + (size_t)scope_index(c, s) * bytes != send)
            CK(cudaMemcpyAsync(rb + (size_t)scope_index(c, s) * bytes, send, bytes, cudaMemcpyDeviceToDevice, c->st));
        return;
    }
    if (c->comm_kind == 3) {   // detached shard: own chunk into every slot (finite, locally timed data)
        for (int j = 0; j < n; ++j)
            if (rb + (size_t)j * bytes != send)
                CK(cudaMemcpyAsync(rb + (size_t)j * bytes, send, bytes, cudaMemcpyDeviceToDevice, c->st));
        return;
    }
    c->timer_begin(T_COMM);
    if (c->comm_kind == 1) {
        NK(ncclAllGather(send, recv, bytes, ncclUint8, scope_comm(c, s), c->st));
    } else {
        LocalGroup& g = *c->lg;
        const std::vector<int> mem = scope_members(c, s);
        const size_t nd = (bytes + 7) / 8;
        if (c->gstage.n < nd) c->gstage.alloc(nd);
        { std::lock_guard<std::mutex> lk(g.m); g.stage[c->rank] = c->gstage.p; }
        CK(cudaMemcpyAsync(c->gstage.p, send, bytes, cudaMemcpyDeviceToDevice, c->st));
        CK(cudaStreamSynchronize(c->st));
        group_barrier(g);
        std::vector<const double*> src;
        {
            std::lock_guard<std::mutex> lk(g.m);
            for (int m : mem) src.push_back(g.stage[m]);
        }
        for (size_t j = 0; j < src.size(); ++j)
            CK(cudaMemcpyAsync(rb + j * bytes, src[j], bytes, cudaMemcpyDefault, c->st));
        CK(cudaStreamSynchronize(c->st));
        group_barrier(g);
    }
    c->timer_end(T_COMM);
}

static void allreduce_sum(Ctx* c, double* buf, size_t n, Scope s = S_ALL) { allreduce(c, buf, n, 0, s); }
static void allreduce_max(Ctx* c, double* buf, size_t n) { allreduce(c, buf, n, 1, S_ALL); }
static void allreduce_max_scope(Ctx* c, double* buf, size_t n, Scope s) { allreduce(c, buf, n, 1, s); }
// view-sharded (partial back projections to sum); a 1-rank NCCL communicator
// on a 2D problem also takes this path (tests the NCCL route bit-exactly)
static bool view_sharded(const Ctx* c) { return c->Rv > 1 || (c->comm_kind == 1 && c->nz == 1); }

static void check_flag(Ctx* c, const char* where) {
    int f = 0;
    CK(cudaMemcpyAsync(&f, c->flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    if (c->fwd3t == 2) {
        int t = 0;
        CK(cudaMemcpyAsync(&t, c->t3flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        if (t) {
            CK(cudaMemsetAsync(c->t3flag.p, 0, sizeof(int), c->st));
            if (t & ~1) throw NumericError(std::string(where) + ": on-the-fly TMA forward: tile/ring error " +
                                           std::to_string(t));
            f |= 1;
        }
    }
    if (f) {
        CK(cudaMemsetAsync(c->flag.p, 0, sizeof(int), c->st));
        std::string what = std::string(where) + ": ";
        if (f & 1) what += "non-finite line integral; ";
        if (f & 2) what += "non-finite AM update; ";
        if (f & 4) what += "non-finite coefficient update; ";
        if (f & 256) what += "fused all-reduce: a peer did not arrive within 10 s; ";
        throw NumericError(what);
    }
}

// ------------------------------------------------------------- system model
static void finish_matrix(Ctx* c, bool have_csc = false) {
    c->zA_L = -1;
    c->band_B = 0; c->band_hb = 0; c->band_P = 0;
    c->blo.release(); c->bhi.release(); c->lacc.release();
    c->phiA_ok = false;
    c->phiA_L = -1;
    for (auto& cm : c->coarse) {
        cm.ok = false;
        cm.rp.release(); cm.cp.release(); cm.col.release(); cm.row.release(); cm.order.release();
        cm.val.release(); cm.valC.release(); cm.cpseg.release(); cm.seg = 1;
    }
    c->phiA_rp.release(); c->phiA_cp.release(); c->phiA_col.release(); c->phiA_row.release();
    c->phiA_val.release(); c->phiA_valC.release(); c->phiA_part.release();
    // CSC mirror (system_matrix.hpp:61-75): stable radix sort of CSR entries by
    // column keeps rows ascending within every column (unless a WAMH v2 cache
    // supplied it: cp and C are then already on the device)
    if (!have_csc) {
    DBuf<unsigned> kin, kout;
    DBuf<uint2> vin, vout;
    kin.alloc(std::max<uint64_t>(c->nnz, 1));
    vin.alloc(std::max<uint64_t>(c->nnz, 1));
    c->cub_tmp.release();
    if (c->nnz) {
        k_csr_to_pairs<<<c->sms * 8, 256, 0, c->st>>>(c->Ml, c->rp.p, c->A.p, kin.p, vin.p);
        check_launch(c, "k_csr_to_pairs");
    }
    sort_pairs(c, kin, vin, kout, vout, c->nnz, c->N);
    kin.release();
    vin.release();
    c->cp.alloc(c->N + 1);
    k_bounds<<<blocks_for(c->N + 1, 256), 256, 0, c->st>>>(kout.p, c->nnz, c->N, c->cp.p);
    check_launch(c, "k_bounds");
    c->C.swap(vout);
    kout.release();
    }
    {   // tiled 2D image layout for the forward gathers: opt-in (WAMGPU_MU_TILED=1).
        // Measured at cfg2 (round 1): 0.773 ms tiled vs 0.7455 ms row-major per
        // forward -- the address arithmetic costs more than the L1 hits it buys.
        const char* e = std::getenv("WAMGPU_MU_TILED");
        const bool want = e && e[0] == '1';
        const bool pow2 = c->nx >= 8 && (c->nx & (c->nx - 1)) == 0 && c->ny % 4 == 0;
        c->lgx = (want && pow2 && c->nz == 1) ? 31 - __builtin_clz((unsigned)c->nx) : -1;
    }
    // C2 compressed forward (2D only), OPT-IN (WAMGPU_C2=1): it halves the
    // forward's DRAM bytes (1.96 vs 3.67 GB at cfg2) but the decode makes it
    // slower (0.81 vs 0.68-0.70 ms, profiles/r01_fwd_patch_sweep.txt), so the
    // uint2 CSR patch forward stays the default
    c->c2_ok = false;
    c->c2_rh.release(); c->c2_codes.release(); c->c2_h.release();
    {
        const char* e = std::getenv("WAMGPU_C2");
        if (c->nz == 1 && c->Ml && e && e[0] == '1' && c->N < (1ull << 30)) {
            DBuf<unsigned long long> nb;
            nb.alloc(c->Ml + 1);
            k_c2_count<<<blocks_for(c->Ml, 256), 256, 0, c->st>>>(c->Ml, c->rp.p, nb.p);
            check_launch(c, "k_c2_count");
            CK(cudaMemsetAsync(nb.p + c->Ml, 0, 8, c->st));
            exclusive_scan_u64(c, nb.p, c->Ml + 1);
            unsigned long long blocks = 0;
            CK(cudaMemcpyAsync(&blocks, nb.p + c->Ml, 8, cudaMemcpyDeviceToHost, c->st));
            CK(cudaStreamSynchronize(c->st));
            c->c2_codes.alloc(std::max<unsigned long long>(blocks, 1) * 8);
            c->c2_rh.alloc(c->Ml);
            c->c2_h.alloc(std::max<unsigned long long>(blocks, 1) * 64);
            CK(cudaMemsetAsync(c->c2_h.p, 0, std::max<unsigned long long>(blocks, 1) * 64 * 4, c->st));
            CK(cudaMemsetAsync(c->c2_codes.p, 0, std::max<unsigned long long>(blocks, 1) * 16, c->st));
            CK(cudaMemsetAsync(c->flag.p, 0, 4, c->st));
            k_c2_build<<<c->sms * 8, 256, 0, c->st>>>(c->Ml, c->rp.p, c->A.p, c->nx, nb.p, c->c2_rh.p,
                                                       c->c2_codes.p, c->c2_h.p, c->flag.p);
            check_launch(c, "k_c2_build");
            int bad = 0;
            CK(cudaMemcpyAsync(&bad, c->flag.p, 4, cudaMemcpyDeviceToHost, c->st));
            CK(cudaMemsetAsync(c->flag.p, 0, 4, c->st));
            CK(cudaStreamSynchronize(c->st));
            c->c2_ok = bad == 0;
            if (!c->c2_ok) { c->c2_rh.release(); c->c2_codes.release(); c->c2_h.release(); }
        }
    }
    c->cub_tmp.release();
    c->nblk_row = (int)std::max<uint64_t>(1, std::min<uint64_t>((c->Ml + 7) / 8, (uint64_t)c->sms * 16));
    c->nblk_col = (int)std::max<uint64_t>(1, std::min<uint64_t>((c->N + 7) / 8, (uint64_t)c->sms * 16));
    c->partial.alloc(std::max<size_t>(std::max(c->nblk_row, 1024), (size_t)c->sms * 16));
    c->scal.alloc(8);
    c->zrow.alloc(c->Ml + 1);
    CK(cudaStreamSynchronize(c->st));
    c->have_matrix = true;
    c->algo = 0;
}

// Sharding.  The ranks form an Rv x Rz grid, rank = zg*Rv + vg:
// view group vg owns the contiguous CSR rows of views [V*vg/Rv, V*(vg+1)/Rv)
// (row = v*D + k, projector.hpp:123-125) and z group zg owns slices
// [nz*zg/Rz, nz*(zg+1)/Rz) (rays never leave their slice, geometry.hpp:17-20).
// A 2D problem shards views only (Rv = R).  An axial 3D stack defaults to
// z-slabs only (Rv = 1, scalars cross GPUs); wamgpu_set_partition picks Rv > 1
// (view shards of a slab sum their partial back projections over comm_v).
// The partition arithmetic itself is host-only (GridPlan), shared with the
// GPU-free wamgpu_plan_partition that the multi-rank CPU tests call.
struct GridPlan {
    int Rv = 1, Rz = 1, vg = 0, zg = 0;
    uint64_t row0 = 0, row1 = 0;
    int s0 = 0, nzl = 1;
};
static GridPlan make_plan(int nz, int views, int detectors, int rank, int R, int vreq) {
    GridPlan p;
    if (R < 1 || rank < 0 || rank >= R) throw ContractError("partition: invalid rank / rank count");
    int Rv = nz == 1 ? R : (vreq > 0 ? vreq : 1);
    if (nz == 1 && vreq > 0 && vreq != R) throw ConfigError("partition: a 2D problem shards views across all ranks");
    if (Rv < 1 || R % Rv) throw ConfigError("partition: view groups must divide the rank count");
    p.Rv = Rv;
    p.Rz = R / Rv;
    p.vg = rank % Rv;
    p.zg = rank / Rv;
    if (nz > 128 * p.Rz) throw ConfigError("wamgpu: at most 128 slices per GPU slab");
    const int v0 = (int)((int64_t)views * p.vg / p.Rv), v1 = (int)((int64_t)views * (p.vg + 1) / p.Rv);
    p.row0 = (uint64_t)v0 * detectors;
    p.row1 = (uint64_t)v1 * detectors;
    if (nz == 1) {
        p.s0 = 0;
        p.nzl = 1;
    } else {
        p.s0 = (int)((int64_t)nz * p.zg / p.Rz);
        p.nzl = (int)((int64_t)nz * (p.zg + 1) / p.Rz) - p.s0;
        if (p.nzl < 1) throw ConfigError("wamgpu: more z groups than slices");
        if (p.nzl > 128) throw ConfigError("wamgpu: at most 128 slices per GPU slab");
    }
    return p;
}

static void resolve_grid(Ctx* c) {
    const GridPlan p = make_plan(c->nz, 1, 1, c->rank, c->nranks, c->vgroups_req);
    c->Rv = p.Rv;
    c->Rz = p.Rz;
    c->vg = p.vg;
    c->zg = p.zg;
    if (c->comm_kind == 1 && c->Rv > 1 && c->Rz > 1 && !c->comm_v) {   // collective over the whole comm
        NK(ncclCommSplit(c->comm, c->zg, c->vg, &c->comm_v, nullptr));
        NK(ncclCommSplit(c->comm, c->vg, c->zg, &c->comm_z, nullptr));
    }
}

static void partition(Ctx* c, int views, int detectors) {
    resolve_grid(c);
    const GridPlan p = make_plan(c->nz, views, detectors, c->rank, c->nranks, c->vgroups_req);
    c->row0 = p.row0;
    c->row1 = p.row1;
    c->s0 = p.s0;
    c->nzl = p.nzl;
    c->Ml = c->row1 - c->row0;
}

static void build_tile_order(Ctx* c) {
    if (c->nz == 1) return;
    std::vector<unsigned> o;
    o.reserve(c->N);
    const int T = 16;
    for (int ty = 0; ty < c->ny; ty += T)
        for (int tx = 0; tx < c->nx; tx += T)
            for (int iy = ty; iy < std::min(ty + T, c->ny); ++iy)
                for (int ix = tx; ix < std::min(tx + T, c->nx); ++ix) o.push_back((unsigned)(iy * c->nx + ix));
    c->order.ensure(c->N);
    CK(cudaMemcpyAsync(c->order.p, o.data(), c->N * 4, cudaMemcpyHostToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));
}

static void set_geometry(Ctx* c, const wamgpu_geometry& g) {
    validate(g);
    std::vector<RayD> rays = ray_table(g);
    c->nx = g.nx; c->ny = g.ny; c->nz = g.nz; c->have_grid = true;
    c->M = (uint64_t)g.views * g.detectors;
    c->N = (uint64_t)g.nx * g.ny;
    partition(c, g.views, g.detectors);
    DBuf<RayDev>& dr = c->rays_dev;   // kept: the on-the-fly forward traces from it
    dr.alloc(std::max<uint64_t>(c->Ml, 1));
    if (c->Ml)
        CK(cudaMemcpyAsync(dr.p, rays.data() + c->row0, c->Ml * sizeof(RayDev), cudaMemcpyHostToDevice, c->st));
    c->geo_D = g.detectors;
    c->geo_V = (int)(c->Ml / (uint64_t)g.detectors);
    c->geo_h = g.voxel_size;
    c->fwd3t = (c->fwd3t_req && c->Ml == (uint64_t)c->geo_V * g.detectors) ? 1 : 0;
    c->t3_cb = 64;
    c->t3_ptr = nullptr;
    c->rp.alloc(c->Ml + 1);
    k_trace_count<<<blocks_for(c->Ml + 1, 128), 128, 0, c->st>>>(dr.p, c->Ml, g.nx, g.ny, g.voxel_size, c->rp.p);
    check_launch(c, "k_trace_count");
    exclusive_scan_u64(c, c->rp.p, c->Ml + 1);
    unsigned long long nnz = 0;
    CK(cudaMemcpyAsync(&nnz, c->rp.p + c->Ml, sizeof(nnz), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    c->nnz = nnz;
    c->A.alloc_padded(std::max<uint64_t>(nnz, 1));
    if (c->Ml) {
        k_trace_fill<<<blocks_for(c->Ml, 128), 128, 0, c->st>>>(dr.p, c->Ml, g.nx, g.ny, g.voxel_size, c->rp.p, c->A.p);
        check_launch(c, "k_trace_fill");
    }
    finish_matrix(c);
    build_tile_order(c);
}

static void set_matrix_csr(Ctx* c, uint64_t rows, uint64_t cols, uint64_t nnz, const uint64_t* rp,
                           const uint32_t* ci, const double* val) {
    if (!rp || (nnz && (!ci || !val))) throw ContractError("SystemMatrix: null array");
    if (rp[0] != 0 || rp[rows] != nnz) throw ContractError("SystemMatrix: inconsistent CSR arrays");
    for (uint64_t y = 0; y < rows; ++y)
        if (rp[y + 1] < rp[y]) throw ContractError("SystemMatrix: row_ptr not monotone");
    if (c->have_grid && (uint64_t)c->nx * c->ny != cols)
        throw ContractError("SystemMatrix: cols != nx*ny of the grid");
    c->M = rows;
    c->N = cols;
    if (!c->have_grid) { c->nx = (int)cols; c->ny = 1; c->nz = 1; }
    // explicit matrices shard by contiguous row blocks (views) and/or z-slab (3D)
    partition(c, (int)rows, 1);
    const uint64_t k0 = rp[c->row0], k1 = rp[c->row1];
    c->nnz = k1 - k0;
    std::vector<unsigned long long> lrp(c->Ml + 1);
    for (uint64_t y = 0; y <= c->Ml; ++y) lrp[y] = rp[c->row0 + y] - k0;
    std::vector<uint2> ent(std::max<uint64_t>(c->nnz, 1));
    for (uint64_t k = 0; k < c->nnz; ++k) {
        if (ci[k0 + k] >= cols) throw ContractError("SystemMatrix: column index out of range");
        ent[k] = make_uint2(ci[k0 + k], 0);
        float f = (float)val[k0 + k];
        std::memcpy(&ent[k].y, &f, 4);
    }
    c->rp.alloc(c->Ml + 1);
    c->A.alloc_padded(std::max<uint64_t>(c->nnz, 1));
    CK(cudaMemcpyAsync(c->rp.p, lrp.data(), (c->Ml + 1) * 8, cudaMemcpyHostToDevice, c->st));
    if (c->nnz) CK(cudaMemcpyAsync(c->A.p, ent.data(), c->nnz * 8, cudaMemcpyHostToDevice, c->st));
    c->rays_dev.release(); c->fwd3t = 0;   // explicit matrix: no ray table to trace from
    finish_matrix(c);
    build_tile_order(c);
}

// ------------------------------------------------------------- WAMH cache
// wamrec::save/load_system_matrix (system_matrix.hpp:87-158).  v1 is the
// reference's layout byte for byte: "WAMH", u32 version = 1, u64 M, N, nnz,
// row_ptr u64[M+1], col_idx u32[nnz], values f64[nnz] (32-byte header, no
// padding).  v2 (this library) stores the device layout so a cache uploads
// without conversion: the v1 header with version = 2, then u64 flags (bit 0:
// CSC mirror present), u32 nx, u32 ny (0 = unknown), row_ptr u64[M+1],
// entries {col u32, h f32}[nnz], and with bit 0 col_ptr u64[N+1] and
// {row u32, h f32}[nnz] (rows ascending per column).  Values on the device
// are fp32 (pin P7), so a v1 file written here carries fp32-representable
// f64 values.  Errors map to IoError like the reference (errors.hpp:32-35).
static constexpr uint64_t WAMH_CHUNK = 1ull << 24;   // entries per streamed chunk

struct File {
    FILE* f = nullptr;
    std::string path;
    File(const char* p, const char* mode) : path(p ? p : "") {
        if (!p) throw ContractError("WAMH: null path");
        f = std::fopen(p, mode);
    }
    ~File() { if (f) std::fclose(f); }
    void read(void* dst, size_t bytes) {
        if (bytes && std::fread(dst, 1, bytes, f) != bytes) throw IoError("unexpected end of file: " + path);
    }
    void write(const void* src, size_t bytes) {
        if (bytes && std::fwrite(src, 1, bytes, f) != bytes) throw IoError("write failed: " + path);
    }
    void seek(uint64_t off) {
        if (fseeko(f, (off_t)off, SEEK_SET) != 0) throw IoError("seek failed: " + path);
    }
    uint64_t size() {
        const off_t cur = ftello(f);
        fseeko(f, 0, SEEK_END);
        const off_t n = ftello(f);
        fseeko(f, cur, SEEK_SET);
        return (uint64_t)n;
    }
};

static void load_matrix_wamh(Ctx* c, const char* path) {
    File F(path, "rb");
    if (!F.f) throw IoError("cannot open for reading: " + F.path);
    char magic[4] = {};
    uint32_t version = 0;
    uint64_t rows = 0, cols = 0, nnz = 0, flags = 0;
    uint32_t gx = 0, gy = 0;
    F.read(magic, 4);
    if (std::memcmp(magic, "WAMH", 4) != 0) throw IoError("not a system-matrix cache file: " + F.path);
    F.read(&version, 4);
    if (version != 1 && version != 2) throw IoError("unsupported cache version in " + F.path);
    F.read(&rows, 8); F.read(&cols, 8); F.read(&nnz, 8);
    uint64_t hdr = 32;
    if (version == 2) { F.read(&flags, 8); F.read(&gx, 4); F.read(&gy, 4); hdr = 48; }
    const bool csc = version == 2 && (flags & 1);
    const uint64_t ebytes = version == 1 ? 12 : 8;
    const uint64_t want = hdr + 8 * (rows + 1) + ebytes * nnz + (csc ? 8 * (cols + 1) + 8 * nnz : 0);
    if (rows > (1ull << 32) || cols > (1ull << 32) || nnz > (1ull << 40) || F.size() != want)
        throw IoError("truncated or inconsistent cache file: " + F.path);
    if (gx && gy) {
        if ((uint64_t)gx * gy != cols) throw IoError("cache grid nx*ny != cols: " + F.path);
        if (c->have_grid && ((uint64_t)c->nx * c->ny != cols)) throw ContractError("WAMH: cols != nx*ny of the grid");
        if (!c->have_grid) { c->nx = (int)gx; c->ny = (int)gy; c->nz = 1; c->have_grid = true; }
    }
    std::vector<uint64_t> rp(rows + 1);
    F.read(rp.data(), 8 * (rows + 1));
    if (rp[0] != 0 || rp[rows] != nnz) throw ContractError("SystemMatrix: inconsistent CSR arrays");
    for (uint64_t y = 0; y < rows; ++y)
        if (rp[y + 1] < rp[y]) throw ContractError("SystemMatrix: row_ptr not monotone");
    if (c->have_grid && (uint64_t)c->nx * c->ny != cols) throw ContractError("SystemMatrix: cols != nx*ny of the grid");
    c->M = rows;
    c->N = cols;
    if (!c->have_grid) { c->nx = (int)cols; c->ny = 1; c->nz = 1; }
    partition(c, (int)rows, 1);
    const uint64_t k0 = rp[c->row0], k1 = rp[c->row1];
    c->nnz = k1 - k0;
    std::vector<unsigned long long> lrp(c->Ml + 1);
    for (uint64_t y = 0; y <= c->Ml; ++y) lrp[y] = rp[c->row0 + y] - k0;
    c->rp.alloc(c->Ml + 1);
    c->A.alloc_padded(std::max<uint64_t>(c->nnz, 1));
    CK(cudaMemcpyAsync(c->rp.p, lrp.data(), (c->Ml + 1) * 8, cudaMemcpyHostToDevice, c->st));
    std::vector<uint2> ent(std::min<uint64_t>(std::max<uint64_t>(c->nnz, 1), WAMH_CHUNK));
    std::vector<uint32_t> ci;
    std::vector<double> val;
    const uint64_t col_off = hdr + 8 * (rows + 1);
    for (uint64_t o = 0; o < c->nnz; o += WAMH_CHUNK) {
        const uint64_t n = std::min(WAMH_CHUNK, c->nnz - o);
        if (version == 1) {   // SoA f64 -> device {col, fp32 h}
            ci.resize(n); val.resize(n);
            F.seek(col_off + 4 * (k0 + o));
            F.read(ci.data(), 4 * n);
            F.seek(col_off + 4 * nnz + 8 * (k0 + o));
            F.read(val.data(), 8 * n);
            for (uint64_t k = 0; k < n; ++k) {
                const float h = (float)val[k];
                ent[k].x = ci[k];
                std::memcpy(&ent[k].y, &h, 4);
            }
        } else {
            F.seek(col_off + 8 * (k0 + o));
            F.read(ent.data(), 8 * n);
        }
        for (uint64_t k = 0; k < n; ++k)
            if (ent[k].x >= cols) throw ContractError("SystemMatrix: column index out of range");
        CK(cudaMemcpy(c->A.p + o, ent.data(), 8 * n, cudaMemcpyHostToDevice));
    }
    // the stored CSC mirror serves only a context holding every row
    const bool use_csc = csc && c->row0 == 0 && c->row1 == rows;
    if (use_csc) {
        const uint64_t csc_off = col_off + 8 * nnz;
        std::vector<unsigned long long> cp(cols + 1);
        F.seek(csc_off);
        F.read(cp.data(), 8 * (cols + 1));
        if (cp[0] != 0 || cp[cols] != nnz) throw IoError("inconsistent CSC mirror in " + F.path);
        c->cp.alloc(cols + 1);
        CK(cudaMemcpyAsync(c->cp.p, cp.data(), 8 * (cols + 1), cudaMemcpyHostToDevice, c->st));
        CK(cudaStreamSynchronize(c->st));
        c->C.alloc_padded(std::max<uint64_t>(nnz, 1));
        for (uint64_t o = 0; o < nnz; o += WAMH_CHUNK) {
            const uint64_t n = std::min(WAMH_CHUNK, nnz - o);
            F.read(ent.data(), 8 * n);
            for (uint64_t k = 0; k < n; ++k)
                if (ent[k].x >= rows) throw ContractError("SystemMatrix: CSC row index out of range");
            CK(cudaMemcpy(c->C.p + o, ent.data(), 8 * n, cudaMemcpyHostToDevice));
        }
    }
    c->rays_dev.release(); c->fwd3t = 0;   // explicit matrix: no ray table to trace from
    finish_matrix(c, use_csc);
    build_tile_order(c);
}

static void save_matrix_wamh(Ctx* c, const char* path, int version, int with_csc) {
    if (!c->have_matrix) throw ContractError("wamgpu: no system matrix set");
    if (version != 1 && version != 2) throw ConfigError("WAMH: version must be 1 or 2");
    if (c->row0 != 0 || c->row1 != c->M)
        throw ContractError("WAMH: this context holds a view shard of the matrix, not all of it");
    File F(path, "wb");
    if (!F.f) throw IoError("cannot open for writing: " + F.path);
    const uint32_t ver = (uint32_t)version;
    const uint64_t M = c->M, N = c->N, nnz = c->nnz;
    F.write("WAMH", 4); F.write(&ver, 4); F.write(&M, 8); F.write(&N, 8); F.write(&nnz, 8);
    const bool csc = version == 2 && with_csc;
    if (version == 2) {
        const uint64_t flags = csc ? 1 : 0;
        const uint32_t gx = c->have_grid && c->nz == 1 ? (uint32_t)c->nx : 0, gy = gx ? (uint32_t)c->ny : 0;
        F.write(&flags, 8); F.write(&gx, 4); F.write(&gy, 4);
    }
    CK(cudaStreamSynchronize(c->st));
    std::vector<unsigned long long> rp(M + 1);
    CK(cudaMemcpy(rp.data(), c->rp.p, 8 * (M + 1), cudaMemcpyDeviceToHost));
    F.write(rp.data(), 8 * (M + 1));
    std::vector<uint2> ent(std::min<uint64_t>(std::max<uint64_t>(nnz, 1), WAMH_CHUNK));
    auto stream = [&](const uint2* dev, uint64_t n_all, auto&& emit) {
        for (uint64_t o = 0; o < n_all; o += WAMH_CHUNK) {
            const uint64_t n = std::min(WAMH_CHUNK, n_all - o);
            CK(cudaMemcpy(ent.data(), dev + o, 8 * n, cudaMemcpyDeviceToHost));
            emit(n);
        }
    };
    if (version == 1) {
        std::vector<uint32_t> ci(ent.size());
        std::vector<double> val(ent.size());
        stream(c->A.p, nnz, [&](uint64_t n) {
            for (uint64_t k = 0; k < n; ++k) ci[k] = ent[k].x;
            F.write(ci.data(), 4 * n);
        });
        stream(c->A.p, nnz, [&](uint64_t n) {
            for (uint64_t k = 0; k < n; ++k) { float h; std::memcpy(&h, &ent[k].y, 4); val[k] = h; }
            F.write(val.data(), 8 * n);
        });
    } else {
        stream(c->A.p, nnz, [&](uint64_t n) { F.write(ent.data(), 8 * n); });
        if (csc) {
            std::vector<unsigned long long> cp(N + 1);
            CK(cudaMemcpy(cp.data(), c->cp.p, 8 * (N + 1), cudaMemcpyDeviceToHost));
            F.write(cp.data(), 8 * (N + 1));
            stream(c->C.p, nnz, [&](uint64_t n) { F.write(ent.data(), 8 * n); });
        }
    }
    if (std::fflush(F.f) != 0) throw IoError("write failed: " + F.path);
}

// ------------------------------------------------------------- pipeline steps
static void need_matrix(Ctx* c) { if (!c->have_matrix) throw ContractError("wamgpu: no system matrix set"); }
static void need_data(Ctx* c) { if (!c->have_data) throw ContractError("wamgpu: no transmission data set"); }

// Slab stride P of the z-fastest 3D layouts: the local slice count rounded up
// to 8, 16, 32, 64 or 128, so a z-slab shard of a few slices (cfg3 on 8 GPUs:
// 8 slices) costs its own slices, not a 32-slice minimum.
static int slab_stride(const Ctx* c) {
    if (c->nzl == 1) return 1;
    int P = 8;
    while (P < c->nzl) P *= 2;
    return P;
}
static int spl_of(const Ctx* c) { return c->nzl <= 32 ? 1 : (c->nzl <= 64 ? 2 : 4); }
static unsigned nblk_warp(const Ctx* c, uint64_t n) {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 7) / 8, (uint64_t)c->sms * 16));
}

// 3D slab SpMM launches (kernels3d.cuh).  WAMGPU_SLAB_VARIANT picks the
// conversion share NF (of 4 values, F2F; the rest by bit moves) of the v2
// kernel:
//   12 = NF 3 (default), 3 = NF 2, 8 = NF 0, 9 = NF 4, 11 = NF 1;
//   1 = round-1 k_forward3/k_back3 (warp per ray, shuffles, F2F only; P >= 32);
//   17 / 18 = NF 3 / 2 with the ping-pong pipeline everywhere, 19 = NF 3 with
//   the copy pipeline everywhere (the round-1 default).  The default runs the
//   ping-pong pipeline (slab_dot_g UX = 104: two register sets, no per-round
//   register copies) in the forward and the plain back projection and the copy
//   pipeline in the fused AM update: cfg4 forward 71.1 -> 64.4, back 61.9 ->
//   56.4 ms per pass; cfg3 8.33 -> 7.62 / 7.73 -> 7.31; cfg5 forward 8.07 ->
//   7.35 but fused-update back 8.01 -> 8.52 (profiles/r06/pp_split_ab.txt).
// Variant + 100 (default 112): the unsigned bit move for vectors known to be
// non-negative.  cfg5 sweep (profiles/r02_slab_sweep.txt): 1 -> 11.3 ms per
// pass, 9 -> 8.45, 12 -> 8.25, 112 -> 8.04 (forward) / 7.89 (back).  One launch
// per 32-slice part (L2-resident part columns at cfg4) was measured slower
// (117 / 111 vs 100 / 70 ms at cfg4) and dropped.
// Lanes per ray by slab stride P: 4 (P = 8, 16: 8 rays per warp), 8 (P = 32,
// 64: 4 rays per warp), 16 (P = 128: 2 rays per warp).
template <int P> struct SlabShape {
    static constexpr int LPR = P <= 16 ? 4 : (P <= 64 ? 8 : 16), SPL = P / LPR, G = 32 / LPR;
};
static int SlabShapeSPL(int P) { return P / (P <= 16 ? 4 : (P <= 64 ? 8 : 16)); }
// X(NF, U, WPB, MINB): F2F share, gathers per round, warps per CTA, min CTAs per SM.
// The default needs MINB = 2: (256, 1) lets ptxas take 170 registers (1 CTA, 8 warps
// per SM) and the slab passes ran 1.65x slower (cfg5 13.5 vs 8.1 ms per forward).
#define SLAB_SWITCH(X, V)                                                                                          \
    switch (V) {                                                                                                   \
        case 3: X(2, 4, 8, 1) break;                                                                               \
        case 8: X(0, 4, 8, 1) break;                                                                               \
        case 9: X(4, 4, 8, 1) break;                                                                               \
        case 11: X(1, 4, 8, 1) break;                                                                              \
        case 13: X(3, 2, 8, 1) break;                                                                              \
        case 14: X(3, 2, 4, 5) break;                                                                              \
        case 15: X(3, 4, 4, 1) break;                                                                              \
        case 16: X(3, 2, 4, 6) break;                                                                              \
        case 17: X(3, 104, 8, 2) break;                                                                            \
        case 18: X(2, 104, 8, 2) break;                                                                            \
        case 20: X(1, 104, 8, 2) break;                                                                            \
        case 21: X(0, 104, 8, 2) break;                                                                            \
        case 19: X(3, 4, 8, 2) break;                                                                              \
        default: X(3, DEFU, 8, 2) break;                                                                           \
    }
// Bands of the 3D forward (k_fwd3s_band): only when the mu slab outgrows L2.
// WAMGPU_FWD_BAND_MB (default 48; 0 = never): target mu bytes per band.
static int forward_bands(Ctx* c) {
    const int P = slab_stride(c);
    if (c->nzl == 1 || !c->Ml) return 1;
    if (c->band_P == P && c->band_B > 0) return c->band_B;
    double mb = 48.0;
    if (const char* e = std::getenv("WAMGPU_FWD_BAND_MB")) mb = std::atof(e);
    const double row = (double)c->nx * P * 4.0, slab = row * c->ny;
    int B = 1, hb = c->ny;
    if (mb > 0.0 && slab > 2.0 * mb * 1048576.0) {
        hb = std::max(1, (int)(mb * 1048576.0 / row));
        B = (c->ny + hb - 1) / hb;
        if (B > 64) { B = 64; hb = (c->ny + B - 1) / B; B = (c->ny + hb - 1) / hb; }
    }
    c->band_P = P;
    c->band_B = B;
    c->band_hb = hb;
    if (B == 1) return 1;
    c->blo.alloc(c->Ml * (uint64_t)B);
    c->bhi.alloc(c->Ml * (uint64_t)B);
    CK(cudaMemsetAsync(c->flag.p, 0, 4, c->st));
    k_band_bounds<<<nblk_warp(c, c->Ml), 256, 0, c->st>>>(c->Ml, c->rp.p, c->A.p, c->nx, hb, B, c->blo.p, c->bhi.p,
                                                          c->flag.p);
    check_launch(c, "k_band_bounds");
    int bad = 0;
    CK(cudaMemcpyAsync(&bad, c->flag.p, 4, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemsetAsync(c->flag.p, 0, 4, c->st));
    CK(cudaStreamSynchronize(c->st));
    if (bad) {   // rows not monotone in iy (explicit matrix): keep the unbanded forward
        c->blo.release(); c->bhi.release();
        c->band_B = 1;
        return 1;
    }
    c->lacc.alloc(c->Ml * (uint64_t)P);
    return B;
}


// ---- on-the-fly 3D forward with TMA-staged tiles (kernels3t.cuh) ----------
// The tensor maps describe the slab vector x[iy][ix][s] (fp32, slab stride P)
// as a 3D tensor (s, ix, iy); boxes of 32 slices x T3_TW x T3_RB pixels for
// x-major bundles and 32 x T3_RB x T3_TW for y-major ones.  The driver entry
// point comes through the runtime (no libcuda link dependency).
typedef CUresult (*PFN_tmEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_tmEncodeTiled tm_encode_fn() {
    static PFN_tmEncodeTiled fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return (PFN_tmEncodeTiled)p;
    }();
    return fn;
}
static bool t3_maps(Ctx* c, const float* x, int P) {
    if (c->t3_ptr == x && c->t3_P == P) return true;
    PFN_tmEncodeTiled enc = tm_encode_fn();
    if (!enc) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)P, (cuuint64_t)c->nx, (cuuint64_t)c->ny};
    const cuuint64_t strides[2] = {(cuuint64_t)P * 4, (cuuint64_t)c->nx * P * 4};
    const cuuint32_t es[3] = {1, 1, 1};
    const cuuint32_t bx[3] = {T3_ZB, T3_TW, T3_RB}, by[3] = {T3_ZB, T3_RB, T3_TW};
    if (enc(&c->t3_mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(x), dims, strides, bx, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    if (enc(&c->t3_my, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(x), dims, strides, by, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    c->t3_ptr = x;
    c->t3_P = P;
    return true;
}
// returns the number of I-divergence partials (CTAs), 0 when the path is not taken.
// Bundle shape: 64 channels x 8 views, or 32 x 16 when the first launch finds a
// 64-channel bundle taller than its tile buffer (wide fans); WAMGPU_FWD3T_NF:
// F2F share of the slab-value conversions (of 4; default 1).
template <int MODE, int NF, int CB>
static void fwd3t_go(Ctx* c, unsigned nb, const T3Args& a, bool uns) {
    static bool attr = false;   // per (MODE, NF, CB)
    if (!attr) {
        CK(cudaFuncSetAttribute(k_fwd3t<MODE, NF, false, CB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(T3Smem)));
        CK(cudaFuncSetAttribute(k_fwd3t<MODE, NF, true, CB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(T3Smem)));
        attr = true;
    }
    if (uns) k_fwd3t<MODE, NF, false, CB><<<nb, T3_RAYS, sizeof(T3Smem), c->st>>>(c->t3_mx, c->t3_my, a);
    else k_fwd3t<MODE, NF, true, CB><<<nb, T3_RAYS, sizeof(T3Smem), c->st>>>(c->t3_mx, c->t3_my, a);
}
template <int MODE>
static unsigned fwd3t_launch(Ctx* c, const float* mu, double* l, bool nonneg) {
    const int P = slab_stride(c);
    if (c->fwd3t <= 0 || P < T3_ZB || !c->rays_dev.p || !c->Ml) return 0;
    if (!t3_maps(c, mu, P)) { c->fwd3t = -1; return 0; }
    const bool uns = nonneg && c->slab_variant >= 100;
    static const int nf = [] { const char* e = std::getenv("WAMGPU_FWD3T_NF"); return e ? std::atoi(e) : 1; }();
    for (;;) {
        const int CB = c->t3_cb, VG = T3_RAYS / CB;
        const unsigned ncb = (c->geo_D + CB - 1) / CB, nvg = (c->geo_V + VG - 1) / VG;
        const unsigned nzc = (c->nzl + T3_ZB - 1) / T3_ZB, nb = ncb * nvg * nzc;
        if (MODE == 1) c->partial.ensure(nb);
        T3Args a{c->rays_dev.p, c->geo_V, c->geo_D, c->nx, c->ny, c->nzl, P, c->geo_h,
                 c->I0.p, c->d.p, c->q.p, l, c->partial.p, c->t3flag.p};
#define T3GO(NFv)                                                          \
    {                                                                      \
        if (CB == 64) fwd3t_go<MODE, NFv, 64>(c, nb, a, uns);              \
        else fwd3t_go<MODE, NFv, 32>(c, nb, a, uns);                       \
    }
        switch (nf) {
            case 0: T3GO(0) break;
            case 2: T3GO(2) break;
            default: T3GO(1) break;
        }
#undef T3GO
        if (c->fwd3t == 2) return nb;
        // first launch for this geometry: did every bundle fit its boxes?
        int f = 0;
        CK(cudaMemcpyAsync(&f, c->t3flag.p, 4, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        if (!(f & ~1)) { c->fwd3t = 2; return nb; }
        CK(cudaMemsetAsync(c->t3flag.p, 0, 4, c->st));
        if (CB == 64 && (f & 0x100)) { c->t3_cb = 32; continue; }   // box too tall (entries then fall outside it): narrower bundles
        std::fprintf(stderr, "[wamgpu] on-the-fly TMA forward rejected for this geometry (flag 0x%x, %d-channel "
                             "bundles): stored-H slab SpMM kept\n", f, CB);
        c->fwd3t = -1;
        return 0;
    }
}

template <int MODE, int P>
static unsigned fwd3_launch_p(Ctx* c, const float* mu, double* l, unsigned maxblk, bool nonneg) {
    using S = SlabShape<P>;
    unsigned nb = 0;
    const int v = c->slab_variant % 100;
    const bool uns = nonneg && c->slab_variant >= 100;
    if constexpr (P >= 32) {
        if (v == 1) {
            nb = std::min<unsigned>(nblk_warp(c, c->Ml), maxblk);
            k_forward3<MODE, P / 32><<<nb, 256, 0, c->st>>>(c->Ml, c->nzl, c->rp.p, c->A.p, mu, c->I0.p, c->d.p,
                                                            c->q.p, l, c->partial.p, c->flag.p);
            return nb;
        }
    }
    const int B = forward_bands(c);
    if (B > 1) {
        // bands in fixed order; MODE 0 accumulates straight in l
        double* acc = MODE == 0 ? l : c->lacc.p;
        nb = std::min<unsigned>(nblk_warp(c, (c->Ml + S::G - 1) / S::G), maxblk);
#define BAND(UXv, SG)                                                                                              \
    k_fwd3s_band<MODE, S::LPR, S::SPL, UXv, 3, SG, P, 8, 2><<<nb, 256, 0, c->st>>>(                                \
        c->Ml, c->nzl, b, B, c->rp.p, c->blo.p, c->bhi.p, c->A.p, mu, c->I0.p, c->d.p, c->q.p, acc, l,             \
        c->partial.p, c->flag.p)
#define BANDN(NFv, SG)                                                                                             \
    k_fwd3s_band<MODE, S::LPR, S::SPL, 104, NFv, SG, P, 8, 2><<<nb, 256, 0, c->st>>>(                              \
        c->Ml, c->nzl, b, B, c->rp.p, c->blo.p, c->bhi.p, c->A.p, mu, c->I0.p, c->d.p, c->q.p, acc, l,             \
        c->partial.p, c->flag.p)
#define BAND2(SG) BANDN(2, SG)
        for (int b = 0; b < B; ++b) {
            if (v == 18 || v == 12) { if (uns) BAND2(false); else BAND2(true); }   // NF 2: cfg4 63.0-63.7 vs 64.1-64.6 ms
            else if (v == 20) { if (uns) BANDN(1, false); else BANDN(1, true); }
            else if (v == 21) { if (uns) BANDN(0, false); else BANDN(0, true); }
            else if (v != 19) { if (uns) BAND(104, false); else BAND(104, true); }
            else { if (uns) BAND(4, false); else BAND(4, true); }
        }
#undef BAND
#undef BAND2
#undef BANDN
        launched(c, B - 1);
        return nb;
    }
#define FX(NF, U, WPB, MINB)                                                                                       \
    {                                                                                                              \
        nb = std::min<unsigned>(nblk_warp(c, (c->Ml + S::G - 1) / S::G) * (8 / WPB), maxblk);                      \
        if (uns)                                                                                                   \
            k_fwd3s<MODE, S::LPR, S::SPL, U, NF, false, P, WPB, MINB><<<nb, 32 * WPB, 0, c->st>>>(                 \
                c->Ml, 0, c->nzl, c->rp.p, c->A.p, mu, c->I0.p, c->d.p, c->q.p, l, c->partial.p, c->flag.p);       \
        else                                                                                                       \
            k_fwd3s<MODE, S::LPR, S::SPL, U, NF, true, P, WPB, MINB><<<nb, 32 * WPB, 0, c->st>>>(                  \
                c->Ml, 0, c->nzl, c->rp.p, c->A.p, mu, c->I0.p, c->d.p, c->q.p, l, c->partial.p, c->flag.p);       \
    }
#define DEFU 104
    SLAB_SWITCH(FX, v)
#undef DEFU
#undef FX
    return nb;
}
// nonneg: the caller guarantees mu >= 0 (AM iterate: mu starts at 0 and every
// update clamps at 0)
template <int MODE>
static unsigned fwd3_launch(Ctx* c, const float* mu, double* l, unsigned maxblk, bool nonneg) {
    unsigned nb = fwd3t_launch<MODE>(c, mu, l, nonneg);
    if (nb) {
        check_launch(c, "k_fwd3t");
        return nb;
    }
    switch (slab_stride(c)) {
        case 8: nb = fwd3_launch_p<MODE, 8>(c, mu, l, maxblk, nonneg); break;
        case 16: nb = fwd3_launch_p<MODE, 16>(c, mu, l, maxblk, nonneg); break;
        case 32: nb = fwd3_launch_p<MODE, 32>(c, mu, l, maxblk, nonneg); break;
        case 64: nb = fwd3_launch_p<MODE, 64>(c, mu, l, maxblk, nonneg); break;
        default: nb = fwd3_launch_p<MODE, 128>(c, mu, l, maxblk, nonneg); break;
    }
    check_launch(c, "k_fwd3s");
    return nb;
}
template <int P>
static void back3_launch_p(Ctx* c, const float* w, double* out, const double* bam, bool nonneg, const TileMap& tm) {
    using S = SlabShape<P>;
    const int v = c->slab_variant % 100;
    const bool uns = nonneg && c->slab_variant >= 100;
    if constexpr (P >= 32) {
        if (v == 1) {
            const unsigned nb = nblk_warp(c, c->N);
            if (bam) k_back3<1, P / 32><<<nb, 256, 0, c->st>>>(c->N, c->nzl, c->order.p, c->cp.p, c->C.p, w, nullptr,
                                                               bam, c->mu.p, c->Z0, c->flag.p);
            else k_back3<0, P / 32><<<nb, 256, 0, c->st>>>(c->N, c->nzl, c->order.p, c->cp.p, c->C.p, w, out,
                                                           nullptr, nullptr, 0.0, c->flag.p);
            return;
        }
    }
#define BX1(NF, U, WPB, MINB, SG)                                                                                  \
    {                                                                                                              \
        const unsigned nb = nblk_warp(c, (c->N + S::G - 1) / S::G) * (8 / WPB);                                    \
        if (bam) k_back3s<1, S::LPR, S::SPL, U, NF, SG, P, WPB, MINB><<<nb, 32 * WPB, 0, c->st>>>(                 \
            c->N, 0, c->nzl, c->order.p, c->cp.p, c->C.p, w, nullptr, bam, c->mu.p, c->Z0, c->flag.p, tm);         \
        else k_back3s<0, S::LPR, S::SPL, U, NF, SG, P, WPB, MINB><<<nb, 32 * WPB, 0, c->st>>>(                     \
            c->N, 0, c->nzl, c->order.p, c->cp.p, c->C.p, w, out, nullptr, nullptr, 0.0, c->flag.p, tm);           \
    }
#define BX(NF, U, WPB, MINB) if (uns) { BX1(NF, U, WPB, MINB, false) } else { BX1(NF, U, WPB, MINB, true) }
    // default: ping-pong pipeline for the plain back projection; the fused AM update keeps the copy
    // pipeline (cfg5: 8.52 vs 8.01 ms per pass with ping-pong)
#define DEFU 104
    if (!bam) {   // default: NF 1 (cfg4 56.3 / 51.3 / 50.1 / 50.4 ms per pass for NF 3 / 2 / 1 / 0, profiles/r06/nf_sweep.txt)
        if (v == 12) { BX(1, 104, 8, 2) } else { SLAB_SWITCH(BX, v) }
    }
#undef DEFU
#define DEFU 4
    if (bam) { SLAB_SWITCH(BX, v) }
#undef DEFU
#undef BX
#undef BX1
}
// nonneg: w >= 0 (the iteration's q and d; not the public back_project)
static void back3_launch(Ctx* c, const float* w, double* out, const double* bam, bool nonneg, const TileMap& tm) {
    switch (slab_stride(c)) {
        case 8: back3_launch_p<8>(c, w, out, bam, nonneg, tm); break;
        case 16: back3_launch_p<16>(c, w, out, bam, nonneg, tm); break;
        case 32: back3_launch_p<32>(c, w, out, bam, nonneg, tm); break;
        case 64: back3_launch_p<64>(c, w, out, bam, nonneg, tm); break;
        default: back3_launch_p<128>(c, w, out, bam, nonneg, tm); break;
    }
}

// g = H^T w (fp64).  2D: CSC gather; 3D: slab gather over the tile-ordered voxels.
// am != nullptr: fused AM update of mu instead of writing g.
// tm (3D only): write g in the tile-major chunk layout of the split update
static void back_launch(Ctx* c, const float* w, double* out, const double* bam, bool nonneg = true,
                        const TileMap& tm = TileMap{}) {
    c->timer_begin(T_BACK);
    if (c->nzl == 1) {
#define BV(U, MB)                                                                                                 \
    if (bam) k_back<1, U, MB><<<c->nblk_col, 256, 0, c->st>>>(c->N, c->cp.p, c->C.p, w, nullptr, bam, c->mu.p,     \
                                                              c->Z0, c->flag.p, c->lgx);                          \
    else k_back<0, U, MB><<<c->nblk_col, 256, 0, c->st>>>(c->N, c->cp.p, c->C.p, w, out, nullptr, nullptr, 0.0,   \
                                                          c->flag.p, -1);
        switch (c->back_variant) {
            case 1: BV(4, 1) break;
            case 2: BV(4, 8) break;
            case 4: BV(8, 6) break;
            case 5: BV(8, 1) break;
#define BP(R, U, MB)                                                                                              \
    if (c->lgx >= 0) throw ConfigError("patch back projection: row-major mu only");                              \
    if (bam) k_back_patch<1, R, U, MB><<<c->nblk_col, 256, 0, c->st>>>(c->N, c->cp.p, c->C.p, w, nullptr, bam,    \
                                                                       c->mu.p, c->Z0, c->flag.p);               \
    else k_back_patch<0, R, U, MB><<<c->nblk_col, 256, 0, c->st>>>(c->N, c->cp.p, c->C.p, w, out, nullptr,        \
                                                                   nullptr, 0.0, c->flag.p);
            case 10: BP(4, 8, 5) break;
            case 11: BP(4, 12, 3) break;
            case 12: BP(2, 8, 5) break;
            case 13: BP(4, 8, 4) break;
            case 14: BP(8, 8, 4) break;
            case 15: BP(2, 12, 3) break;
#undef BP
            default: BV(12, 1) break;     // measured best at cfg2 (round 1 sweep, profiles/)
        }
#undef BV
    } else {
        back3_launch(c, w, out, bam, nonneg, tm);
    }
    check_launch(c, "k_back3");
    c->timer_end(T_BACK);
    c->tm.back_launches++;
    c->tm.proj_updates += (int64_t)(c->nnz * (uint64_t)c->nzl);
}
// nonneg: w >= 0 with no -0.0 (q, d); false for caller-supplied vectors
static void back_into(Ctx* c, const float* w, double* out, bool nonneg = true) {
    back_launch(c, w, out, nullptr, nonneg);
}

// one cooperative launch of the fused back projection + all-reduce (kernels_ar.cuh);
// rexec logical ranks [a.r0, a.r0 + rexec) run in this grid
template <class Prod>
static void launch_fused_ar(int sms, cudaStream_t st, ArArgs a, const Prod& prod, int rexec) {
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fused_allreduce<Prod>, 256, 0));
    const uint64_t ntiles = (a.n + AR_TILE - 1) / AR_TILE;
    const int per = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)per_sm * sms / rexec, ntiles));
    if (per * rexec > per_sm * sms) throw ConfigError("fused all-reduce: ranks exceed the co-resident CTAs");
    a.rexec = rexec;
    Prod p = prod;
    void* args[] = {&a, &p};
    CK(cudaLaunchCooperativeKernel((void*)k_fused_allreduce<Prod>, dim3(per * rexec), dim3(256), args, 0, st));
}

// [g || extra] = sum over ranks of (H_r^T w || extra_r): one fused kernel per
// rank; the result is left in c->ar.res (n = 2N) on every rank
static void back_allreduce(Ctx* c, const float* w, const double* extra) {
    c->timer_begin(T_BACK);
    ArProdBack pb{};
    pb.cp[c->rank] = c->cp.p;
    pb.C[c->rank] = c->C.p;
    pb.w[c->rank] = w;
    pb.extra[c->rank] = extra;
    pb.N = c->N;
    ArArgs a = c->ar.args;
    a.epoch = ++c->ar.args.epoch;
    a.r0 = c->rank;
    a.err = c->flag.p;
    launch_fused_ar(c->sms, c->st, a, pb, 1);
    check_launch(c, "k_fused_allreduce");
    c->timer_end(T_BACK);
    c->tm.back_launches++;
    c->tm.proj_updates += (int64_t)(c->nnz * (uint64_t)c->nzl);
}

// plain l = H mu (fp64 out), for forward_project
static void forward_plain(Ctx* c, const float* mu, double* l) {
    if (c->nzl == 1) {
        if (c->lgx >= 0)
            k_forward<0, FG_DEFAULT, 8, 1, true><<<c->nblk_row, 256, 0, c->st>>>(c->Ml, c->rp.p, c->A.p, mu, nullptr,
                                                                              nullptr, nullptr, l, nullptr, c->flag.p,
                                                                              c->lgx);
        else if (c->c2_ok)
            k_fwd_c2<0, 5><<<c->nblk_row, 256, 0, c->st>>>(c->Ml, c->rp.p, c->c2_rh.p, c->c2_codes.p, c->c2_h.p,
                                                          c->nx, mu, nullptr, nullptr, nullptr, l, nullptr, c->flag.p);
        else
            k_fwd_patch<0, 4, 8, 5><<<c->nblk_row, 256, 0, c->st>>>(c->Ml, c->rp.p, c->A.p, mu, nullptr, nullptr,
                                                                   nullptr, l, nullptr, c->flag.p);
    } else {
        fwd3_launch<0>(c, mu, l, nblk_warp(c, c->Ml), false);
    }
    check_launch(c, "k_forward3");
}

static int coarse_k(const Ctx* c);
static int coarse_mode();
static unsigned fwd2c_launch(Ctx* c, int k);
static unsigned fwd3c_launch(Ctx* c, int k, unsigned maxblk);
static void sync_mu(Ctx* c);
// q = I0 exp(-H mu), objective -> scal[0] (all-reduced), record
static void forward_fused(Ctx* c, bool record) {
    const int ck = c->algo == 2 ? coarse_k(c) : 0;
    c->timer_begin(ck > 0 ? T_FWDC : T_FWD);
    int nparts = c->nblk_row;
    uint64_t entries = c->nnz, slices = (uint64_t)c->nzl;
    if (c->nzl == 1 && ck > 0) {
        nparts = (int)fwd2c_launch(c, ck);
        entries = c->coarse[ck].nnz;
    } else if (c->nzl == 1) {
#define FV(FGv, U, MB)                                                                                              \
    if (c->lgx >= 0)                                                                                               \
        k_forward<1, FGv, U, MB, true><<<c->nblk_row, 256, 0, c->st>>>(c->Ml, c->rp.p, c->A.p, c->mu.p, c->I0.p,    \
                                                                    c->d.p, c->q.p, nullptr, c->partial.p,         \
                                                                    c->flag.p, c->lgx);                            \
    else                                                                                                           \
        k_forward<1, FGv, U, MB, false><<<c->nblk_row, 256, 0, c->st>>>(c->Ml, c->rp.p, c->A.p, c->mu.p, c->I0.p,   \
                                                                     c->d.p, c->q.p, nullptr, c->partial.p,        \
                                                                     c->flag.p, -1);
        switch (c->fwd_variant) {
            case 1: FV(1, 8, 1) break;
            case 2: FV(2, 4, 1) break;
            case 3: FV(2, 4, 6) break;
            case 5: FV(2, 12, 1) break;
            case 6: FV(4, 4, 1) break;
            case 7: FV(1, 8, 6) break;
            case 8: FV(2, 8, 1) break;
#define FP(R, U, MB)                                                                                               \
    k_fwd_patch<1, R, U, MB><<<c->nblk_row, 256, 0, c->st>>>(c->Ml, c->rp.p, c->A.p, c->mu.p, c->I0.p, c->d.p,      \
                                                            c->q.p, nullptr, c->partial.p, c->flag.p);
            case 10: FP(4, 4, 8) break;
            case 11: FP(4, 8, 4) break;
            case 12: FP(2, 4, 8) break;
            case 13: FP(8, 4, 8) break;
            case 14: FP(4, 6, 6) break;
            case 15: FP(8, 8, 4) break;
            case 16: FP(4, 2, 8) break;
            case 17: FP(4, 12, 3) break;
            case 18: FP(4, 8, 5) break;
            case 19: FP(2, 8, 4) break;
            case 20: FP(4, 16, 2) break;
            case 21: FP(4, 10, 4) break;
            case 22: FP(8, 12, 3) break;
            case 23: FP(4, 8, 6) break;
            case 24: FP(8, 8, 5) break;
            case 25: FP(4, 6, 5) break;
            case 26: FP(2, 8, 5) break;
            case 9: FV(1, 4, 8) break;    // round-1 default (row-per-warp)
#define FC2(MB)                                                                                                  \
    if (c->c2_ok) k_fwd_c2<1, MB><<<c->nblk_row, 256, 0, c->st>>>(c->Ml, c->rp.p, c->c2_rh.p, c->c2_codes.p,       \
                                                                  c->c2_h.p, c->nx, c->mu.p, c->I0.p, c->d.p,     \
                                                                  c->q.p, nullptr, c->partial.p, c->flag.p);      \
    else FP(4, 8, 5)
            case 40: FC2(4) break;
            case 41: FC2(6) break;
            case 42: FC2(8) break;
            default: FC2(5) break;        // C2 when built (WAMGPU_C2=1), else FP(4,8,5): the measured best
#undef FC2
        }
#undef FP
#undef FV
    } else {
        if (ck > 0) {
            nparts = (int)fwd3c_launch(c, ck, (unsigned)c->partial.n);
            entries = c->coarse[ck].nnz;
            if (coarse_mode() >= 2) slices = (uint64_t)(c->nzl >> ck);
        }
        else nparts = (int)fwd3_launch<1>(c, c->mu.p, nullptr, (unsigned)c->partial.n, c->algo == 1 && c->mu_nonneg);
    }
    check_launch(c, "k_forward3");
    c->timer_end(ck > 0 ? T_FWDC : T_FWD);
    if (ck > 0) c->tm.coarse_fwd_launches++; else c->tm.fwd_launches++;
    c->tm.proj_updates += (int64_t)(entries * slices);
    k_sum_partials<<<1, 1024, 0, c->st>>>(c->partial.p, nparts, c->scal.p);
    check_launch(c, "k_sum_partials");
    allreduce_sum(c, c->scal.p, 1);
    if (record) {
        k_record<<<1, 32, 0, c->st>>>(c->scal.p, c->counters.p, c->objs.p, c->cums.p, c->it.p);
        check_launch(c, "k_record");
    }
}

static double device_max(Ctx* c, const double* v, uint64_t n) {
    const int nb = (int)std::min<uint64_t>(std::max<uint64_t>(1, (n + 255) / 256), 1024);
    k_max_partials<<<nb, 256, 0, c->st>>>(v, n, c->partial.p);
    check_launch(c, "k_max_partials");
    k_max_partials<<<1, 256, 0, c->st>>>(c->partial.p, (uint64_t)nb, c->scal.p + 1);
    check_launch(c, "k_max_partials");
    allreduce_max(c, c->scal.p + 1, 1);
    double m = 0.0;
    CK(cudaMemcpyAsync(&m, c->scal.p + 1, 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    return m;
}

static void launch_walk(Ctx* c, int L) {
    const unsigned nb = blocks_for(c->Ml + 1, 32 * WALK_WARPS);
#define WALK_CASE(LV)                                                                                        \
    case LV:                                                                                                 \
        k_walk<LV><<<nb, 32 * WALK_WARPS, 0, c->st>>>(c->Ml, c->rp.p, c->A.p, c->nx,                        \
                                                      c->haar3 ? cpow3_host(LV) : 1.0, c->zA.p, c->zrow.p); \
        break;
    switch (L) {
        WALK_CASE(0) WALK_CASE(1) WALK_CASE(2) WALK_CASE(3) WALK_CASE(4) WALK_CASE(5)
        default: throw ConfigError("haar: depth beyond the device walk");
    }
#undef WALK_CASE
    check_launch(c, "k_walk");
}


static void upload_tree_bits(Ctx* c, const std::vector<uint8_t>& src) {
    // host tree bytes -> bit-packed, levels at 32-bit aligned bit offsets
    std::vector<unsigned> w;
    uint64_t bit = 0;
    for (int l = 0; l <= LMAX + 1; ++l) c->boff.off[l] = 0;
    for (int l = 1; l <= c->L; ++l) {
        const uint64_t n = (uint64_t)(c->nx >> l) * (c->ny >> l);
        const uint8_t* a = src.data() + c->off.off[l];
        bool any = false;   // levels without bits are never looked up: not uploaded
        for (uint64_t i = 0; i < n && !any; ++i) any = a[i] != 0;
        if (!any) continue;
        c->boff.off[l] = bit;
        w.resize((bit + n + 31) / 32 + 1, 0u);
        for (uint64_t i = 0; i < n; ++i)
            if (a[i]) w[(bit + i) >> 5] |= 1u << ((bit + i) & 31);
        bit = (bit + n + 31) / 32 * 32;
    }
    if (w.empty()) w.push_back(0u);
    c->tree_words = (int)w.size();
    c->tbits.ensure(w.size());
    CK(cudaMemcpyAsync(c->tbits.p, w.data(), w.size() * 4, cudaMemcpyHostToDevice, c->st));
}

// incremental expansion walk over the new-block bits in tbits: levels in
// lvpack (4 bits each, nlev warps), zfix -> zfix2, triples -> kin_s / vin_s
static void launch_walk_lv(Ctx* c, int nlev, unsigned lvpack, unsigned long long cap,
                           unsigned long long* kcnt = nullptr) {
    // G ray groups of 32 per CTA so that a CTA has ~4 warps whatever nlev is
    const int G = std::max(1, 4 / nlev);
    const unsigned nb = blocks_for(c->Ml, 32 * G);
#define WL(D, NS)                                                                                                 \
    {                                                                                                             \
        const size_t smem = walk_smem(G, nlev, c->tree_words, D, NS).total;                                       \
        if (smem > 200 * 1024) throw ConfigError("tree too large for the shared-memory walk");                    \
        CK(cudaFuncSetAttribute(k_walk_lv<D, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));       \
        k_walk_lv<D, NS><<<nb, 32 * nlev * G, smem, c->st>>>(c->Ml, c->rp.p, c->A.p, c->nx, c->ny, nlev, G, lvpack, \
                                                            c->tbits.p, c->boff, c->tree_words, c->zfix.p,        \
                                                            c->zfix2.p, c->cursor.p, cap, c->kin_s.p, c->vin_s.p,  \
                                                            kcnt);                                                \
    }
    switch (c->walk_variant) {
        case 1: WL(8, 2) break;
        case 2: WL(16, 2) break;
        case 3: WL(32, 1) break;
        case 4: WL(4, 2) break;
        default: WL(16, 1) break;   // measured best at cfg2 (expand 17.6 ms vs 19.0 for (8,2))
    }
#undef WL
    check_launch(c, "k_walk_lv");
}


// ---- separable 3D Haar (pin P3) helpers -------------------------------------
static uint64_t blocks2(const Ctx* c, int l) { return (uint64_t)(c->nx >> l) * (c->ny >> l); }
static int zwords(const Ctx* c, int l) { return ((c->nzl >> l) + 31) >> 5; }

// act_host (3D bytes, level l: (nzl>>l, ny>>l, nx>>l)) -> any-bits per in-plane
// block (shared memory of the walk) + z-activity words per in-plane block.
template <class Fn>
static void host_par_chunks(uint64_t n, uint64_t align, Fn&& fn);

static void upload_tree3(Ctx* c, int* nlev_out) {
    std::vector<unsigned> w, zw;
    uint64_t bit = 0, zo = 0, ko = 0;
    for (int l = 0; l <= LMAX + 1; ++l) c->boff.off[l] = c->zoff.off[l] = c->koff.off[l] = 0;
    int nlev = 0, fine = 0;
    bool chain = true;
    std::vector<uint2> lst;
    for (int l = c->L; l >= 1; --l) {
        const uint64_t nb = blocks2(c, l);
        const int nk = c->nzl >> l, W = zwords(c, l);
        c->boff.off[l] = bit;
        c->zoff.off[l] = zo;
        c->koff.off[l] = ko;
        w.resize((bit + nb + 31) / 32 + 1, 0u);
        zw.resize(zo + nb * W, 0u);
        const uint8_t* a = c->act_host.data() + c->off.off[l];
        // parallel over in-plane block ranges aligned to 32 (each thread owns
        // its tbits words and its blocks' z words); lists concatenate in order
        std::vector<std::vector<uint2>> parts;
        std::mutex pm;
        std::atomic<bool> any_l{false};
        host_par_chunks(nb, 32, [&](uint64_t lo, uint64_t hi, int t) {
            bool any = false;
            for (int k = 0; k < nk; ++k) {
                const uint8_t* ak = a + (uint64_t)k * nb;
                for (uint64_t b = lo; b < hi; ++b)
                    if (ak[b]) {
                        zw[zo + b * W + (k >> 5)] |= 1u << (k & 31);
                        w[(bit + b) >> 5] |= 1u << ((bit + b) & 31);
                        any = true;
                    }
            }
            std::vector<uint2> mine;
            for (uint64_t b = lo; b < hi; ++b)
                if ((w[(bit + b) >> 5] >> ((bit + b) & 31)) & 1u) mine.push_back(make_uint2((unsigned)b, (unsigned)l));
            std::lock_guard<std::mutex> lk(pm);
            if ((int)parts.size() <= t) parts.resize(t + 1);
            parts[t].swap(mine);
            if (any) any_l = true;
        });
        // The split gathers one q row per Psi entry and every block's list spans all
        // views.  In row-major block order the blocks in flight cover a few full image
        // rows, i.e. nearly every ray: the q slab (cfg4: 755 MB) streams from DRAM again
        // and again (ncu: 222 GB per launch, 27% L2 hits).  Morton order keeps the blocks
        // in flight inside a compact square.  (The split writes by block index, so the
        // order is free.)  WAMGPU_SPLIT_ORDER=0: row-major.
        static const int split_order = [] { const char* e = std::getenv("WAMGPU_SPLIT_ORDER"); return e ? std::atoi(e) : 1; }();
        if (split_order == 1) {
            if (c->morton_nx != c->nx || c->morton_ny != c->ny) {
                c->morton.clear();
                c->morton_nx = c->nx; c->morton_ny = c->ny;
            }
            if ((int)c->morton.size() <= l) c->morton.resize(l + 1);
            std::vector<unsigned>& perm = c->morton[l];
            if (perm.size() != nb) {   // once per grid and level
                const unsigned wl = (unsigned)(c->nx >> l);
                auto spread = [](uint64_t v) {
                    v = (v | (v << 16)) & 0x0000ffff0000ffffull;
                    v = (v | (v << 8)) & 0x00ff00ff00ff00ffull;
                    v = (v | (v << 4)) & 0x0f0f0f0f0f0f0f0full;
                    v = (v | (v << 2)) & 0x3333333333333333ull;
                    v = (v | (v << 1)) & 0x5555555555555555ull;
                    return v;
                };
                std::vector<std::pair<uint64_t, unsigned>> kv(nb);
                for (uint64_t b = 0; b < nb; ++b) kv[b] = {spread(b % wl) | (spread(b / wl) << 1), (unsigned)b};
                std::sort(kv.begin(), kv.end());
                perm.resize(nb);
                for (uint64_t b = 0; b < nb; ++b) perm[b] = kv[b].second;
            }
            for (uint64_t i = 0; i < nb; ++i) {
                const uint64_t b = perm[i];
                if ((w[(bit + b) >> 5] >> ((bit + b) & 31)) & 1u) lst.push_back(make_uint2((unsigned)b, (unsigned)l));
            }
        } else {
            for (auto& v : parts) lst.insert(lst.end(), v.begin(), v.end());
        }
        if (any_l) fine = l;   // levels run L..1: the last hit is the finest
        if (chain && any_l) ++nlev; else chain = false;
        bit = (bit + nb + 31) / 32 * 32;
        zo += nb * W;
        ko += nb;
    }
    if (w.empty()) w.push_back(0u);
    if (zw.empty()) zw.push_back(0u);
    c->tree_words = (int)w.size();
    c->nkeys3 = ko;
    c->tbits.ensure(w.size());
    c->zbits.ensure(zw.size());
    CK(cudaMemcpyAsync(c->tbits.p, w.data(), w.size() * 4, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->zbits.p, zw.data(), zw.size() * 4, cudaMemcpyHostToDevice, c->st));
    c->fine_level = fine;
    c->nlist3 = lst.size();
    c->list3.ensure(std::max<size_t>(lst.size(), 1));
    if (!lst.empty()) CK(cudaMemcpyAsync(c->list3.p, lst.data(), lst.size() * 8, cudaMemcpyHostToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));
    *nlev_out = std::max(nlev, 1);
}

template <int MODE>
static void launch_walk3h(Ctx* c, int nlev, unsigned long long* cnt, const unsigned long long* pos) {
    const unsigned nb = blocks_for(c->Ml, 32);
    // shared memory: the per-(ray, z-block) totals of the WALKED levels (Z walk only)
    size_t stot = 0;
    if (MODE == 1)
        for (int l = c->L; l > c->L - nlev && l >= 1; --l) stot += (size_t)(c->nzl >> l) * 32 * 8;
    const size_t smem = stot;
    if (smem > 200 * 1024) throw ConfigError("slab too deep for the shared-memory 3D walk");
    // Z walk with level 1 walked and >= 32 level-1 z-blocks: a second warp
    // takes half of the level-1 flush loop (WAMGPU_WALK3_SPLIT=0 turns it off)
    static const bool split_on = [] {
        const char* e = std::getenv("WAMGPU_WALK3_SPLIT");
        return !(e && e[0] == '0');
    }();
    const int split1 = (MODE == 1 && split_on && nlev == c->L && (c->nzl >> 1) >= 32) ? 1 : 0;
#define W3(LV)                                                                                                   \
    case LV: {                                                                                                   \
        auto kf = k_walk3h<MODE, LV>;                                                                            \
        if (smem > 32 * 1024) CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        kf<<<nb, 32 * (nlev + split1), smem, c->st>>>(c->Ml, c->rp.p, c->A.p, c->nx, c->ny, c->nzl, c->tbits.p,  \
                                           c->boff, c->tree_words, c->zbits.p, c->zoff, c->koff, c->zA.p, c->zrow.p, \
                                           cnt, pos, c->kin_s.p, c->vin_s.p, c->pray_s.p, c->ppsi_s.p, split1);    \
    } break;
    switch (c->L) {
        W3(1) W3(2) W3(3) W3(4) W3(5)
        default: throw ConfigError("haar3: depth beyond the device walk");
    }
#undef W3
    check_launch(c, "k_walk3h");
}

// Psi lists (per in-plane block with any active z-block): count -> scan ->
// emit -> stable radix sort by key -> payload gather -> CSC by key.
static void rebuild_psi3(Ctx* c, int nlev) {
    const uint64_t ncnt = (uint64_t)c->Ml * c->L;
    CK(cudaMemsetAsync(c->wcnt.p + ncnt, 0, 8, c->st));
    exclusive_scan_u64(c, c->wcnt.p, ncnt + 1);
    unsigned long long tot = 0;
    CK(cudaMemcpyAsync(&tot, c->wcnt.p + ncnt, 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    const uint64_t n1 = std::max<uint64_t>(tot, 1);
    c->kin_s.ensure(n1); c->vin_s.ensure(n1); c->pray_s.ensure(n1); c->ppsi_s.ensure(n1);
    if (tot) launch_walk3h<2>(c, nlev, nullptr, c->wcnt.p);
    HTRACE("expand3: Psi count scan + emit walk");
    // persistent sort output: a per-call buffer meant a GB-sized cudaMalloc +
    // cudaFree (which synchronizes) in every expansion
    DBuf<uint2>& sidx = c->sidx3;
    sort_pairs(c, c->kin_s, c->vin_s, c->kout_s, sidx, tot, c->nkeys3);
    HTRACE("expand3: Psi sort");
    c->E3ray.ensure_padded(n1);
    c->E3psi.ensure_padded(n1);
    if (tot) {
        k_gather_psi<<<blocks_for(tot, 256), 256, 0, c->st>>>(tot, sidx.p, c->pray_s.p, c->ppsi_s.p, c->E3ray.p,
                                                               c->E3psi.p);
        check_launch(c, "k_gather_psi");
    }
    c->np.ensure(c->nkeys3 + 1);
    k_bounds<<<blocks_for(c->nkeys3 + 1, 256), 256, 0, c->st>>>(c->kout_s.p, tot, c->nkeys3, c->np.p);
    check_launch(c, "k_bounds");
    c->nnz_phi = tot;
    // ray bands of the split (WAMGPU_SPLIT_BAND_MB; default 0 = off: measured no
    // gain, cfg4 52.4-55.5 vs 53.0 ms per launch, profiles/r06/pp_split_ab.txt): only
    // when the q slab outgrows L2
    {
        static const double mb = [] { const char* e = std::getenv("WAMGPU_SPLIT_BAND_MB"); return e ? std::atof(e) : 0.0; }();
        const double row = (double)slab_stride(c) * 4.0, slab = row * (double)c->Ml;
        int B = 1;
        unsigned rpb = (unsigned)c->Ml;
        if (mb > 0.0 && tot && slab > 2.0 * mb * 1048576.0) {
            rpb = (unsigned)std::max(1.0, mb * 1048576.0 / row);
            B = (int)((c->Ml + rpb - 1) / rpb);
            if (B > 32) { B = 32; rpb = (unsigned)((c->Ml + B - 1) / B); B = (int)((c->Ml + rpb - 1) / rpb); }
        }
        c->sband_B = B;
        if (B > 1) {
            const uint64_t n = c->nkeys3 * (uint64_t)(B + 1);
            c->bptr3.ensure(n);
            k_split_band_ptr<<<blocks_for(n, 256), 256, 0, c->st>>>(c->nkeys3, c->np.p, c->E3ray.p, B, rpb, c->bptr3.p);
            check_launch(c, "k_split_band_ptr");
        }
    }
    CK(cudaStreamSynchronize(c->st));
}

// Z0 = max_y sum_{z active} |phi(y|z)| (Eq. 1.61).  init: the approximation part
// (tree-independent, cached in zA); AM: levels = 0 -> row sums.
// (The 2D tree's Z(y) is kept incrementally in fixed point by phi_append; the
// non-init path here is the separable 3D model's.)
static double compute_z0(Ctx* c, int levels, bool init) {
    c->zA.ensure(c->Ml + 1);
    if (init) {
        // zA depends only on (matrix, levels, Haar model, local rows): like
        // the CSC and Phi_A it is computed once per matrix and reused by later
        // inits (finish_matrix drops it)
        if (c->Ml && c->zA_L == levels && c->zA_h3 == c->haar3 && c->zA_r0 == c->row0 && c->zA_Ml == c->Ml) {
            CK(cudaMemcpyAsync(c->zrow.p, c->zA.p, c->Ml * sizeof(double), cudaMemcpyDeviceToDevice, c->st));
        } else if (c->Ml) {
            launch_walk(c, levels);
            c->zA_L = levels; c->zA_h3 = c->haar3; c->zA_r0 = c->row0; c->zA_Ml = c->Ml;
        }
    } else if (c->Ml && c->haar3) {
        c->wcnt.ensure((uint64_t)c->Ml * std::max(levels, 1) + 1);
        int nlev = 1;
        upload_tree3(c, &nlev);
        c->walk_nlev = nlev;
        launch_walk3h<1>(c, nlev, c->wcnt.p, nullptr);
    } else if (c->Ml) {
        throw std::logic_error("compute_z0: the 2D tree keeps Z(y) incrementally (zfix)");
    }
    double z0 = device_max(c, c->zrow.p, c->Ml);
    if (!(z0 > 0.0)) throw NumericError("Z0: no ray intersects the active set");
    return z0;
}

static void ensure_records(Ctx* c, int n) {
    if ((int)c->objs.n < n) {
        c->objs.alloc(n);
        c->cums.alloc(n);
    }
    CK(cudaMemsetAsync(c->it.p, 0, sizeof(int), c->st));
    while ((int)c->ev_iter.size() < n) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        c->ev_iter.push_back(e);
    }
}

static void begin_call(Ctx* c) {
    c->tm = wamgpu_timing{};
    for (int k = 0; k < T_NCAT; ++k) c->tev_used[k] = 0;
    c->launches = 0;
    CK(cudaEventRecord(c->ev_a, c->st));
}

static void end_call(Ctx* c) {
    CK(cudaEventRecord(c->ev_b, c->st));
    CK(cudaEventSynchronize(c->ev_b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev_a, c->ev_b));
    c->tm.total_ms = ms;
    double* dst[T_NCAT] = {&c->tm.fwd_ms, &c->tm.back_ms, &c->tm.split_ms, &c->tm.update_ms, &c->tm.expand_ms,
                           &c->tm.comm_ms, &c->tm.phi_ms, &c->tm.coarse_fwd_ms, &c->tm.coarse_back_ms};
    for (int k = 0; k < T_NCAT; ++k) {
        double s = 0.0;
        for (size_t i = 0; i < c->tev_used[k]; ++i) {
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, c->tev[k][i].first, c->tev[k][i].second));
            s += t;
        }
        *dst[k] = s;
    }
    c->tm.kernel_launches = c->launches;
    c->tm.split_nnz = (int64_t)c->nnz_phi;
}

static void fill_records(Ctx* c, int n, wamgpu_record* recs, int64_t active_at_start) {
    if (!recs) return;
    std::vector<double> o(n);
    std::vector<unsigned long long> cu(n);
    CK(cudaMemcpyAsync(o.data(), c->objs.p, n * 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(cu.data(), c->cums.p, n * 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    for (int i = 0; i < n; ++i) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, c->ev_t0, c->ev_iter[i]));
        recs[i].iter = c->iter - n + i + 1;
        recs[i].objective = o[i];
        recs[i].elapsed_s = ms * 1e-3;
        recs[i].active_set = active_at_start;
        recs[i].cum_updates = (int64_t)cu[i];
    }
}

// ---- boundary layout conversion: reference image/coefficient layout
// ((s0+s)*N + x, image.hpp:14) <-> device slab [x][s]; rays (s*M + y) <-> [y][s].

// host-side data-parallel loop for the boundary conversions (large 3D slabs)
template <class Fn>
static void host_par(uint64_t n, Fn&& fn) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const uint64_t nt = n < (1u << 20) ? 1 : std::min<uint64_t>(hw, 32);
    if (nt == 1) { fn(0, n); return; }
    std::vector<std::thread> pool;
    const uint64_t chunk = (n + nt - 1) / nt;
    for (uint64_t t = 0; t < nt; ++t) {
        const uint64_t lo = t * chunk, hi = std::min(n, lo + chunk);
        if (lo < hi) pool.emplace_back([&fn, lo, hi] { fn(lo, hi); });
    }
    for (auto& th : pool) th.join();
}
// chunks aligned to `align` elements, fn(lo, hi, chunk index); serial below 64K
template <class Fn>
static void host_par_chunks(uint64_t n, uint64_t align, Fn&& fn) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const uint64_t nt = n < (1u << 16) ? 1 : std::min<uint64_t>(hw, 16);
    if (nt == 1) { fn(0, n, 0); return; }
    const uint64_t chunk = ((n + nt - 1) / nt + align - 1) / align * align;
    std::vector<std::thread> pool;
    for (uint64_t t = 0; t * chunk < n; ++t) {
        const uint64_t lo = t * chunk, hi = std::min(n, lo + chunk);
        pool.emplace_back([&fn, lo, hi, t] { fn(lo, hi, (int)t); });
    }
    for (auto& th : pool) th.join();
}
// number of bytes set in a[lo, hi) minus those set in b (host, parallel)
static int64_t count_diff(const uint8_t* a, const uint8_t* b, uint64_t n) {
    std::atomic<int64_t> tot{0};
    host_par_chunks(n, 64, [&](uint64_t lo, uint64_t hi, int) {
        int64_t s = 0;
        for (uint64_t i = lo; i < hi; ++i) s += (a[i] != 0) - (b ? (b[i] != 0) : 0);
        tot += s;
    });
    return tot.load();
}

static uint64_t NV(const Ctx* c) { return c->N * (uint64_t)slab_stride(c); }
static uint64_t MV(const Ctx* c) { return c->Ml * (uint64_t)slab_stride(c); }
// 2D image upload/download through the tiled device layout (mu_addr)
static void upload_image2(Ctx* c, const double* ref, float* dev) {
    std::vector<float> h(c->N);
    for (uint64_t x = 0; x < c->N; ++x) h[mu_addr((unsigned)x, c->lgx)] = (float)ref[x];
    CK(cudaMemcpyAsync(dev, h.data(), c->N * 4, cudaMemcpyHostToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));
}
static void download_image2(Ctx* c, const float* dev, double* ref) {
    std::vector<float> h(c->N);
    CK(cudaMemcpyAsync(h.data(), dev, c->N * 4, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    for (uint64_t x = 0; x < c->N; ++x) ref[x] = h[mu_addr((unsigned)x, c->lgx)];
}

// Streamed host<->device transfers through two pinned 32 MB staging buffers:
// the host fills (drains) one while the other is in flight.  The strided
// reference<->slab reorder runs on the device (k_ref_to_slab / k_slab_to_ref);
// the host only converts contiguous runs between double and the device type.
constexpr size_t kPinChunk = 32u << 20;
static void ensure_pinned(Ctx* c) {
    if (c->pin[0]) return;
    for (int k = 0; k < 2; ++k) {
        CK(cudaMallocHost(&c->pin[k], kPinChunk));
        CK(cudaEventCreateWithFlags(&c->pin_ev[k], cudaEventDisableTiming));
    }
}
// fill(h, lo, hi): write elements [lo, hi) of the host-side sequence to h[0 ..)
template <class T, class Fill>
static void h2d_streamed(Ctx* c, T* dev, uint64_t count, Fill&& fill) {
    ensure_pinned(c);
    const uint64_t per = kPinChunk / sizeof(T);
    int k = 0;
    for (uint64_t lo = 0; lo < count; lo += per, k ^= 1) {
        const uint64_t hi = std::min(count, lo + per);
        CK(cudaEventSynchronize(c->pin_ev[k]));   // this buffer's previous copy has left
        T* h = static_cast<T*>(c->pin[k]);
        host_par(hi - lo, [&](uint64_t a, uint64_t b) { fill(h + a, lo + a, lo + b); });
        CK(cudaMemcpyAsync(dev + lo, h, (hi - lo) * sizeof(T), cudaMemcpyHostToDevice, c->st));
        CK(cudaEventRecord(c->pin_ev[k], c->st));
    }
}
// drain(h, lo, hi): consume elements [lo, hi) of the device sequence from h[0 ..)
template <class T, class Drain>
static void d2h_streamed(Ctx* c, const T* dev, uint64_t count, Drain&& drain) {
    ensure_pinned(c);
    const uint64_t per = kPinChunk / sizeof(T);
    const uint64_t nch = (count + per - 1) / per;
    auto issue = [&](uint64_t ch) {
        const uint64_t lo = ch * per, hi = std::min(count, lo + per);
        CK(cudaMemcpyAsync(c->pin[ch & 1], dev + lo, (hi - lo) * sizeof(T), cudaMemcpyDeviceToHost, c->st));
        CK(cudaEventRecord(c->pin_ev[ch & 1], c->st));
    };
    if (nch) issue(0);
    for (uint64_t ch = 0; ch < nch; ++ch) {
        if (ch + 1 < nch) issue(ch + 1);           // its buffer was drained in the previous round
        CK(cudaEventSynchronize(c->pin_ev[ch & 1]));
        const uint64_t lo = ch * per, hi = std::min(count, lo + per);
        const T* h = static_cast<const T*>(c->pin[ch & 1]);
        host_par(hi - lo, [&](uint64_t a, uint64_t b) { drain(h + a, lo + a, lo + b); });
    }
}

template <class T>
static void upload_slab(Ctx* c, const double* ref, T* dev, uint64_t n_inner, uint64_t ref_stride, uint64_t ref_off,
                        bool local = false) {
    const int P = slab_stride(c);
    const int sb = local ? 0 : c->s0;
    const int nzl = c->nzl;
    const uint64_t count = (uint64_t)nzl * n_inner;
    c->xfer.ensure(std::max<uint64_t>(count, 1) * sizeof(T));
    T* xs = reinterpret_cast<T*>(c->xfer.p);
    h2d_streamed<T>(c, xs, count, [&](T* h, uint64_t lo, uint64_t hi) {
        uint64_t s = lo / n_inner, i = lo % n_inner;
        const double* r = ref + (uint64_t)(sb + s) * ref_stride + ref_off;
        for (uint64_t e = lo; e < hi; ++e) {
            *h++ = (T)r[i];
            if (++i == n_inner) { i = 0; ++s; r = ref + (uint64_t)(sb + s) * ref_stride + ref_off; }
        }
    });
    if (n_inner) {
        k_ref_to_slab<T><<<dim3((unsigned)((n_inner + 31) / 32), (unsigned)((P + 31) / 32)), dim3(32, 8), 0, c->st>>>(
            xs, dev, n_inner, nzl, P);
        check_launch(c, "k_ref_to_slab");
    }
    CK(cudaStreamSynchronize(c->st));
}
template <class T>
static void download_slab(Ctx* c, const T* dev, double* ref, uint64_t n_inner, uint64_t ref_stride, uint64_t ref_off,
                          bool local = false) {
    const int P = slab_stride(c);
    const int sb = local ? 0 : c->s0;
    const int nzl = c->nzl;
    const uint64_t count = (uint64_t)nzl * n_inner;
    c->xfer.ensure(std::max<uint64_t>(count, 1) * sizeof(T));
    T* xs = reinterpret_cast<T*>(c->xfer.p);
    if (n_inner) {
        k_slab_to_ref<T><<<dim3((unsigned)((n_inner + 31) / 32), (unsigned)((P + 31) / 32)), dim3(32, 8), 0, c->st>>>(
            dev, xs, n_inner, nzl, P);
        check_launch(c, "k_slab_to_ref");
    }
    d2h_streamed<T>(c, xs, count, [&](const T* h, uint64_t lo, uint64_t hi) {
        uint64_t s = lo / n_inner, i = lo % n_inner;
        double* r = ref + (uint64_t)(sb + s) * ref_stride + ref_off;
        for (uint64_t e = lo; e < hi; ++e) {
            r[i] = (double)*h++;
            if (++i == n_inner) { i = 0; ++s; r = ref + (uint64_t)(sb + s) * ref_stride + ref_off; }
        }
    });
}

// ------------------------------------------------------------------ AM
static void am_init(Ctx* c, const double* init_mu) {
    need_matrix(c);
    need_data(c);
    c->mu.ensure(NV(c));
    c->g.ensure(2 * NV(c));
    c->bam.ensure(NV(c));
    // the AM update clamps at +0, so mu stays sign-bit-free when
    // it starts so: the 3D forward may then use the unsigned bit move
    c->mu_nonneg = true;
    if (init_mu) {
        for (uint64_t i = 0; i < c->N * (uint64_t)c->nz && c->mu_nonneg; ++i) c->mu_nonneg = !std::signbit(init_mu[i]);
        if (c->nzl == 1) upload_image2(c, init_mu, c->mu.p);
        else upload_slab<float>(c, init_mu, c->mu.p, c->N, c->N, 0);
    } else {
        CK(cudaMemsetAsync(c->mu.p, 0, NV(c) * 4, c->st));
    }
    back_into(c, c->d.p, c->bam.p);  // b(x) = sum_y d(y) h(y|x)
    if (view_sharded(c)) allreduce_sum(c, c->bam.p, NV(c), S_VIEWS);
    if (!c->act.p) { c->act.alloc(1); }
    c->Z0 = compute_z0(c, 0, true);  // Z0 = max_y sum_x h(y|x)
    forward_fused(c, false);
    CK(cudaMemsetAsync(c->counters.p, 0, 16, c->st));
    CK(cudaEventRecord(c->ev_t0, c->st));
    check_flag(c, "am_init");
    c->algo = 1;
    c->iter = 0;
    c->active = (int64_t)c->N * c->nz;
}

// View groups of a 3D slab (Rv > 1) can split the update instead of
// replicating it: reduce-scatter the partial back projections by image rows,
// update only the member's rows (AM) or tile rows (3D Haar), all-gather the
// result.  Moves 24 instead of 32 bytes per coefficient (WAM) and 12 instead of
// 16 (AM) through the collective, and divides the update by Rv.
// WAMGPU_VIEW_UPDATE=allreduce keeps the all-reduce + replicated update.
static bool split_update_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("WAMGPU_VIEW_UPDATE");
        return !(e && std::strcmp(e, "allreduce") == 0);
    }();
    return on;
}
static bool am_split_update(const Ctx* c) {
    return c->nz > 1 && c->Rv > 1 && split_update_enabled() && c->ny % c->Rv == 0;
}
static bool wam_split_update(const Ctx* c) {
    return c->nz > 1 && c->haar3 && c->Rv > 1 && split_update_enabled() && ((c->ny >> c->L) % c->Rv) == 0;
}
static TileMap make_tilemap(const Ctx* c) {
    TileMap m;
    m.L = c->L;
    m.TX = c->nx >> c->L;
    m.TZ = c->nzl >> c->L;
    m.rows = (c->ny >> c->L) / c->Rv;
    m.nx = c->nx;
    m.ny = c->ny;
    m.nzl = c->nzl;
    m.CT = (uint64_t)m.rows * m.TX * m.TZ << (3 * c->L);
    return m;
}

static void am_iterate(Ctx* c, int n, wamgpu_record* recs) {
    if (c->algo != 1) throw ContractError("am: not initialised");
    ensure_records(c, n);
    for (int i = 0; i < n; ++i) {
        if (!view_sharded(c)) {
            back_launch(c, c->q.p, nullptr, c->bam.p);   // fused multiplicative update
        } else {
            const double* g = c->g.p;
            if (am_split_update(c)) {   // 3D view group: reduce-scatter g, own rows, all-gather mu
                back_into(c, c->q.p, c->g.p);
                const uint64_t CA = NV(c) / c->Rv, o = CA * c->vg;
                c->rs_recv.ensure(CA);
                reduce_scatter(c, c->g.p, c->rs_recv.p, CA, S_VIEWS);
                k_am_update<<<blocks_for(CA, 256), 256, 0, c->st>>>(CA, c->rs_recv.p, c->bam.p + o, c->mu.p + o,
                                                                     c->Z0, c->flag.p, -1);
                check_launch(c, "k_am_update");
                all_gather(c, c->mu.p + o, c->mu.p, CA * 4, S_VIEWS);
                CK(cudaMemsetAsync(c->counters.p, 0, 8, c->st));
                forward_fused(c, true);
                CK(cudaEventRecord(c->ev_iter[i], c->st));
                c->iter++;
                continue;
            }
            if (c->ar.on && c->nz == 1) {   // fused back projection + all-reduce over NVLink peer memory
                back_allreduce(c, c->q.p, c->ar.extra.p);   // extra = zeros here
                g = c->ar.res.p;
            } else {
                back_into(c, c->q.p, c->g.p);
                allreduce_sum(c, c->g.p, NV(c), S_VIEWS);
            }
            k_am_update<<<blocks_for(NV(c), 256), 256, 0, c->st>>>(NV(c), g, c->bam.p, c->mu.p, c->Z0, c->flag.p,
                                                                    c->nz == 1 ? c->lgx : -1);
            check_launch(c, "k_am_update");
        }
        CK(cudaMemsetAsync(c->counters.p, 0, 8, c->st));
        forward_fused(c, true);
        CK(cudaEventRecord(c->ev_iter[i], c->st));
        c->iter++;
    }
    check_flag(c, "am_iterate");
    if (recs) {
        std::vector<double> o(n);
        CK(cudaMemcpyAsync(o.data(), c->objs.p, n * 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        for (int i = 0; i < n; ++i) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, c->ev_t0, c->ev_iter[i]));
            recs[i].iter = c->iter - n + i + 1;
            recs[i].objective = o[i];
            recs[i].elapsed_s = ms * 1e-3;
            recs[i].active_set = c->active;
            recs[i].cum_updates = c->active * recs[i].iter;
        }
    }
}

// ------------------------------------------------------------------ WAM
static void tile_launch(Ctx* c, int mode, double* mu64, double* out) {
    const int TS = 1 << c->L;
    if (c->haar3) {
        dim3 grid(c->nx >> c->L, c->ny >> c->L, c->nzl >> c->L);
        const size_t smem = 2ull * TS * TS * TS * sizeof(double);
        if (smem > 48 * 1024)
            CK(cudaFuncSetAttribute(k_tile3h, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_tile3h<<<grid, 256, smem, c->st>>>(mode, c->nx, c->ny, c->nzl, slab_stride(c), c->L, c->g.p, c->g.p + NV(c),
                                             c->bdata.p, c->act.p, c->off, c->beta.p, c->mu.p, mu64, out, c->bp_dbg.p,
                                             c->bm_dbg.p, c->Z0, c->counters.p, c->flag.p);
        check_launch(c, "k_tile3h");
        return;
    }
    if (c->nzl == 1) {
        dim3 grid(c->nx >> c->L, c->ny >> c->L);
        const int bs = std::min(1024, std::max(32, TS * TS));
        const size_t smem = 2ull * TS * TS * sizeof(double);
        k_tile<<<grid, bs, smem, c->st>>>(mode, c->nx, c->ny, c->L, c->g.p, c->g.p + c->N, c->bdata.p, c->act.p,
                                          c->off, c->beta.p, c->mu.p, mu64, out, c->bp_dbg.p, c->bm_dbg.p, c->Z0,
                                          c->counters.p, c->flag.p, c->lgx);
    } else {
        const int sc = std::max(1, std::min({32, c->nzl, 4096 / (TS * TS)}));   // slices per CTA
        dim3 grid(c->nx >> c->L, c->ny >> c->L, (c->nzl + sc - 1) / sc);
        const size_t smem = 2ull * sc * TS * TS * sizeof(double);
        if (smem > 48 * 1024)
            CK(cudaFuncSetAttribute(k_tile3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_tile3<<<grid, 256, smem, c->st>>>(mode, c->nx, c->ny, c->nzl, slab_stride(c), c->L, sc, c->g.p, c->g.p + NV(c), c->bdata.p,
                                            c->act.p, c->off, c->beta.p, c->mu.p, mu64, out, c->bp_dbg.p,
                                            c->bm_dbg.p, c->Z0, c->counters.p, c->flag.p);
    }
    check_launch(c, "k_tile3");
}

// Z0 = max_y Z(y) from the fixed-point rows (zrow receives the doubles)
static void z0_from_zfix(Ctx* c) {
    if (c->Ml) {
        k_zfix_to_d<<<blocks_for(c->Ml, 256), 256, 0, c->st>>>(c->Ml, c->zfix.p, c->zrow.p);
        check_launch(c, "k_zfix_to_d");
    }
    const double z0 = device_max(c, c->zrow.p, c->Ml);
    if (!(z0 > 0.0)) throw NumericError("Z0: no ray intersects the active set");
    c->Z0 = z0;
}

// Bring Phi^- (CSC over local rays, active details) and Z(y) up to the current
// tree act_host from the tree act_phi they cover.  Columns of blocks that were
// already active never change: one walk over the NEW blocks (k_walk_lv) emits
// their negative phi as unsorted triples and adds their |phi| terms to the
// fixed-point Z.  The batch is placed by COUNTING straight into E after the
// existing entries: the walk takes the key histogram as it drains its lane
// rings (sentinel entries are not counted), an exclusive scan gives the column
// bounds, and k_key_place moves each entry to its column's cursor
// (warp-aggregated).  WAMGPU_PHI_SORT=1 keeps the older path, a CUB radix sort
// by key.  k_cols_set records each new column's [lo, hi).  Within a column the
// ray order is arbitrary: the split sums in exact fixed point.

static void phi_append(Ctx* c) {
    // active detail list from the host tree (level by level, the H, V, D of a
    // block adjacent: the split is order-free and they share rays), new bits
    std::vector<unsigned> lst;
    std::vector<uint8_t> nw(c->act_bytes, 0);
    bool lv_new[LMAX + 2] = {};
    for (int l = 1; l <= c->L; ++l) {
        const int wl = c->nx >> l, hl = c->ny >> l;
        const uint64_t o = c->off.off[l];
        const uint8_t* a = c->act_host.data() + o;
        for (int bi = 0; bi < hl; ++bi)
            for (int bj = 0; bj < wl; ++bj) {
                const uint64_t i = (uint64_t)bi * wl + bj;
                if (!a[i]) continue;
                lst.push_back((unsigned)((hl + bi) * c->nx + bj));
                lst.push_back((unsigned)(bi * c->nx + wl + bj));
                lst.push_back((unsigned)((hl + bi) * c->nx + wl + bj));
                if (!c->act_phi[o + i]) { nw[o + i] = 1; lv_new[l] = true; }
            }
    }
    HTRACE("expand: list + new bits");
    c->nlist = lst.size();
    c->list.ensure(std::max<size_t>(lst.size(), 1));
    if (!lst.empty())
        CK(cudaMemcpyAsync(c->list.p, lst.data(), lst.size() * 4, cudaMemcpyHostToDevice, c->st));
    int nlev = 0;
    unsigned lvpack = 0;
    for (int l = c->L; l >= 1; --l)
        if (lv_new[l]) { lvpack |= (unsigned)l << (4 * nlev); ++nlev; }
    if (nlev == 0 || c->Ml == 0) {
        c->act_phi = c->act_host;
        if (nlev) z0_from_zfix(c);   // collective: every rank takes part
        CK(cudaStreamSynchronize(c->st));
        return;
    }
    upload_tree_bits(c, nw);
    HTRACE("expand: list/tree upload");
    c->cursor.ensure(1);
    c->zfix2.ensure(c->Ml + 1);
    // capacity guess for the batch (a short guess costs a second walk)
    unsigned long long tot = 0;
    uint64_t cap = std::max<uint64_t>({c->kin_s.n, 2 * c->phi_batch, c->nnz / 4, (uint64_t)1 << 20});
    static const bool use_sort = [] {
        const char* e = std::getenv("WAMGPU_PHI_SORT");
        return e && e[0] == '1';
    }();
    c->ptmp.ensure(c->N + 1);
    for (int attempt = 0;; ++attempt) {
        c->kin_s.ensure(cap);
        c->vin_s.ensure(cap);
        CK(cudaMemsetAsync(c->cursor.p, 0, 8, c->st));
        if (!use_sort) CK(cudaMemsetAsync(c->ptmp.p, 0, (c->N + 1) * 8, c->st));
        launch_walk_lv(c, nlev, lvpack, c->kin_s.n, use_sort ? nullptr : c->ptmp.p);
        CK(cudaMemcpyAsync(&tot, c->cursor.p, 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        if (tot <= c->kin_s.n) break;
        if (attempt) throw NumericError("phi-: emission count changed between walks");
        cap = tot + tot / 8;
    }
    c->phi_batch = tot;
    HTRACE("expand: walk");
    // append: E keeps the first nnz_phi entries, the sorted batch follows
    const uint64_t off = c->nnz_phi;
    if (c->E.n < off + tot + 64) {
        DBuf<uint2> t;
        t.alloc(off + tot + (off + tot) / 2 + 64);
        if (off) CK(cudaMemcpyAsync(t.p, c->E.p, off * sizeof(uint2), cudaMemcpyDeviceToDevice, c->st));
        c->E.swap(t);
    }
    c->ptmp.ensure(c->N + 1);
    HTRACE("expand: E grow");
    // Counting placement (default): the walk histogrammed the batch's keys
    // into ptmp (sentinels not counted), exclusive scan into the column
    // bounds, warp-aggregated placement.  WAMGPU_PHI_SORT=1 keeps the earlier
    // radix sort + k_bounds (same runs, other ray order).
    if (!use_sort) {
        exclusive_scan_u64(c, c->ptmp.p, c->N + 1);
        if (tot) {
            c->pcur.ensure(c->N + 1);
            CK(cudaMemcpyAsync(c->pcur.p, c->ptmp.p, (c->N + 1) * 8, cudaMemcpyDeviceToDevice, c->st));
            k_key_place<<<blocks_for(tot, 256), 256, 0, c->st>>>(tot, c->kin_s.p, c->vin_s.p, (unsigned)c->N,
                                                                   c->pcur.p, c->E.p + off);
            check_launch(c, "k_key_place");
        }
        HTRACE("expand: place");
    } else {
    c->kout_s.ensure(std::max<uint64_t>(tot, 1));
    if (tot) {
        const int bits = bits_for(c->N);
        auto vi = reinterpret_cast<unsigned long long*>(c->vin_s.p);
        auto vo = reinterpret_cast<unsigned long long*>(c->E.p + off);
        size_t tb = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, c->kin_s.p, c->kout_s.p, vi, vo, (int64_t)tot, 0, bits,
                                           c->st));
        c->cub_tmp.ensure(tb + 1);
        CK(cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tb, c->kin_s.p, c->kout_s.p, vi, vo, (int64_t)tot, 0, bits,
                                           c->st));
        launched(c, 4);
    }
    HTRACE("expand: sort");
    k_bounds<<<blocks_for(c->N + 1, 256), 256, 0, c->st>>>(c->kout_s.p, tot, c->N, c->ptmp.p);
    check_launch(c, "k_bounds");
    }
    k_cols_set<<<blocks_for(c->N, 256), 256, 0, c->st>>>(c->N, c->ptmp.p, off, c->cols.p);
    check_launch(c, "k_cols_set");
    // ptmp[N] = the batch's valid entries: the scan total on the counting path
    // (sentinels never counted), the sentinel key N's bound on the sort path
    unsigned long long valid = 0;
    CK(cudaMemcpyAsync(&valid, c->ptmp.p + c->N, 8, cudaMemcpyDeviceToHost, c->st));
    c->zfix.swap(c->zfix2);
    z0_from_zfix(c);
    c->nnz_phi = off + valid;
    c->act_phi = c->act_host;
    HTRACE("expand: bounds + Z0");
}

static int64_t count_active(const Ctx* c) {
    if (c->haar3) {
        // levels 1..L are contiguous in act_host (wam_init): 7 details per set byte
        const int64_t a = (int64_t)(c->nx >> c->L) * (c->ny >> c->L) * (c->nzl >> c->L);
        return a + 7 * count_diff(c->act_host.data(), nullptr, c->act_bytes);
    }
    int64_t a = (int64_t)(c->nx >> c->L) * (c->ny >> c->L);
    for (int l = 1; l <= c->L; ++l) {
        const uint64_t n = (uint64_t)(c->nx >> l) * (c->ny >> l);
        const uint8_t* p = c->act_host.data() + c->off.off[l];
        for (uint64_t i = 0; i < n; ++i) a += 3 * (p[i] != 0);
    }
    return a * c->nz;
}

static void split_init(Ctx* c);
static bool phiA_applicable(const Ctx* c);
static void build_phiA(Ctx* c);

static void wam_init(Ctx* c, int L, const double* init_beta) {
    need_matrix(c);
    need_data(c);
    if (!c->have_grid) throw ContractError("wam: image grid unknown (set_geometry or set_grid)");
    if (L < 0 || L > LMAX) throw ConfigError("haar: depth must be in [0, " + std::to_string(LMAX) + "]");
    if ((c->nx % (1 << L)) || (c->ny % (1 << L))) throw ConfigError("haar: slice dimensions not divisible by 2^L");
    if (c->haar3 && (c->nzl % (1 << L) || c->s0 % (1 << L)))
        throw ConfigError("haar3: the slab's slices must be divisible by 2^L (and slab-aligned)");
    if (c->haar3 && L < 1) throw ConfigError("haar3: depth must be >= 1");
    c->L = L;
    const uint64_t N = NV(c);  // local slab of coefficients / voxels
    c->mu.ensure(N); c->beta.ensure(N); c->g.ensure(2 * N); c->bdata.ensure(N); c->mu64.ensure(N);
    c->bp_dbg.ensure(N); c->bm_dbg.ensure(N);
    CK(cudaMemsetAsync(c->g.p, 0, 2 * N * 8, c->st));
    CK(cudaMemsetAsync(c->bp_dbg.p, 0, N * 8, c->st));
    CK(cudaMemsetAsync(c->bm_dbg.p, 0, N * 8, c->st));
    // tree bitmaps, level l at off[l]
    uint64_t o = 0;
    for (int l = 0; l <= LMAX + 1; ++l) c->off.off[l] = 0;
    for (int l = 1; l <= L; ++l) {
        c->off.off[l] = o;
        o += (uint64_t)(c->nx >> l) * (c->ny >> l) * (c->haar3 ? (uint64_t)(c->nzl >> l) : 1);
    }
    c->act_bytes = o;
    c->act.ensure(std::max<uint64_t>(o, 1));
    c->act_new.ensure(std::max<uint64_t>(o, 1));
    CK(cudaMemsetAsync(c->act.p, 0, std::max<uint64_t>(o, 1), c->st));
    c->act_host.assign(o, 0);
    if (init_beta) {
        upload_slab<float>(c, init_beta, c->beta.p, c->N, c->N, 0);
    } else {
        CK(cudaMemsetAsync(c->beta.p, 0, N * 4, c->st));
    }
    // b(z) = [Omega^T H^T d](z) for every z
    back_into(c, c->d.p, c->g.p);
    if (view_sharded(c)) allreduce_sum(c, c->g.p, N, S_VIEWS);
    tile_launch(c, 2, nullptr, c->bdata.p);
    CK(cudaMemsetAsync(c->g.p, 0, 2 * N * 8, c->st));
    if (c->ar.extra.p) CK(cudaMemsetAsync(c->ar.extra.p, 0, c->N * 8, c->st));   // fused path: no stale b-
    c->Z0 = compute_z0(c, L, true);
    c->nlist = 0;
    c->nlist3 = 0;
    c->fine_level = 0;
    c->mu_c_k = -1;
    c->stats_k = -1;
    c->nnz_phi = 0;
    c->phi_batch = 0;
    if (!c->haar3) {                     // 3D: the tree is empty, no Psi lists yet
        // empty tree: Z(y) = F(zA(y)) in fixed point, Phi^- empty
        c->zfix.ensure(c->Ml + 1);
        if (c->Ml) {
            k_zfix_init<<<blocks_for(c->Ml, 256), 256, 0, c->st>>>(c->Ml, c->zA.p, c->zfix.p);
            check_launch(c, "k_zfix_init");
        }
        z0_from_zfix(c);
        c->cols.ensure(c->N);
        CK(cudaMemsetAsync(c->cols.p, 0, c->N * sizeof(ulonglong2), c->st));
        c->act_phi.assign(c->act_bytes, 0);
    }
    tile_launch(c, 0, nullptr, nullptr);  // mu = Omega beta
    c->mu_stale = false;
    c->bown_stale = false;
    c->phiA_beta_ok = init_beta == nullptr;   // Φ_A covers the roots only: inactive details must be 0
    if (phiA_applicable(c)) build_phiA(c);
    split_init(c);
    forward_fused(c, false);
    CK(cudaMemsetAsync(c->counters.p, 0, 16, c->st));
    CK(cudaEventRecord(c->ev_t0, c->st));
    check_flag(c, "wam_init");
    c->algo = 2;
    c->iter = 0;
    c->active = count_active(c);
}

// ---- Φ_A projections while the tree holds only the approximation roots ----
constexpr int kPhiSeg = 8;
static bool phiA_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("WAMGPU_PHI_A");
        return !(e && e[0] == '0');
    }();
    return on;
}
// slices per lane of the 3D Φ_A kernels (lane-owned slices stay in one z-block)
static int phiA3_spl(const Ctx* c) { return std::max(1, slab_stride(c) / 32); }
static bool phiA_applicable(const Ctx* c) {
    if (!phiA_enabled() || c->L < 1 || !c->phiA_beta_ok) return false;
    if (c->nz == 1) return !c->haar3;
    return c->haar3 && phiA3_spl(c) <= (1 << c->L);   // separable 3D Haar (pin P3)
}
// CSR by ray (count, scan, fill) and CSC by coefficient (stable key sort)
static void build_phiA(Ctx* c) {
    if (c->phiA_ok && c->phiA_L == c->L) return;
    c->phiA_ok = false;
    c->phiA_rp.alloc(c->Ml + 1);
    k_phiA_count<<<blocks_for(c->Ml + 1, 128), 128, 0, c->st>>>(c->Ml, c->rp.p, c->A.p, c->nx, c->L, c->phiA_rp.p);
    check_launch(c, "k_phiA_count");
    exclusive_scan_u64(c, c->phiA_rp.p, c->Ml + 1);
    unsigned long long nnz = 0;
    CK(cudaMemcpyAsync(&nnz, c->phiA_rp.p + c->Ml, 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    const uint64_t n1 = std::max<unsigned long long>(nnz, 1);
    c->phiA_col.alloc(n1);
    c->phiA_val.alloc(n1);
    DBuf<unsigned> kin, kout;
    DBuf<uint2> vin, vout;
    kin.alloc(n1);
    vin.alloc(n1);
    k_phiA_fill<<<blocks_for(c->Ml, 128), 128, 0, c->st>>>(c->Ml, c->rp.p, c->A.p, c->nx, c->L, c->phiA_rp.p,
                                                            c->phiA_col.p, c->phiA_val.p, kin.p, vin.p);
    check_launch(c, "k_phiA_fill");
    sort_pairs(c, kin, vin, kout, vout, nnz, c->N);
    kin.release();
    vin.release();
    c->phiA_row.alloc(n1);
    c->phiA_valC.alloc(n1);
    if (nnz) {
        k_phiA_gather<<<blocks_for(nnz, 256), 256, 0, c->st>>>(nnz, vout.p, c->phiA_val.p, c->phiA_row.p,
                                                              c->phiA_valC.p);
        check_launch(c, "k_phiA_gather");
    }
    c->phiA_cp.alloc(c->N + 1);
    k_bounds<<<blocks_for(c->N + 1, 256), 256, 0, c->st>>>(kout.p, nnz, c->N, c->phiA_cp.p);
    check_launch(c, "k_bounds");
    const uint64_t nA = (uint64_t)(c->nx >> c->L) * (c->ny >> c->L);
    const uint64_t NK = c->haar3 ? (uint64_t)(c->nzl >> c->L) : 1;
    c->phiA_part.alloc(nA * kPhiSeg * NK);
    if (c->haar3) c->phiA_mblk.alloc(nA * NK);
    CK(cudaStreamSynchronize(c->st));
    c->phiA_nnz = nnz;
    c->phiA_L = c->L;
    c->phiA_ok = true;
}
// ---- block-coarsened projections (kernels3c.cuh) ---------------------------
// WAMGPU_COARSE=0: always project over H.  WAMGPU_COARSE_CHECK=1: verify on
// the device, before every coarse forward, that mu is constant on the blocks.
// WAMGPU_COARSE: 0 = always project over H; 1 = in-plane blocks only; 2 (default) = in-plane
// blocks and z-groups.  Read per call: tests switch it between contexts.
static int coarse_mode() {
    const char* e = std::getenv("WAMGPU_COARSE");
    return e ? std::atoi(e) : 2;
}
static bool coarse_enabled() { return coarse_mode() != 0; }
static bool coarse_root() {   // default on: cfg4 12.69 -> 13.17 it/s, cfg3 71.4 -> 74.7 (profiles/r07/root_ab.txt)
    const char* e = std::getenv("WAMGPU_COARSE_ROOT");
    return !(e && e[0] == '0');
}
static int pow2_stride(int n) {
    int P = 8;
    while (P < n) P *= 2;
    return P;
}
// coarsening exponent k (block edge 2^k) the current tree allows; 0 = project over H
static int coarse_k(const Ctx* c) {
    // view shards: each rank coarsens its own rows; the partial [g || b-] are all-reduced after the
    // expansion to pixels.  Not with the fused NVLink all-reduce (2D) or the split update (3D view
    // groups), whose back projections write other layouts.
    if (!coarse_enabled() || !c->phiA_beta_ok || c->ar.on || wam_split_update(c)) return 0;
    const bool d3 = c->haar3 && c->nzl > 1, d2 = !c->haar3 && c->nz == 1 && c->lgx < 0;
    if (!d3 && !d2) return 0;   // (the per-slice 2D Haar model of a 3D stack keeps the pixel path)
    // root-only tree (no detail active): 2^L cubes.  3D only (WAMGPU_COARSE_ROOT=0: the Phi_A
    // iteration of kernels_phi.cuh instead); the 2D root-only phase always runs over Phi_A.
    if (c->fine_level == 0 && !(d3 && coarse_root() && coarse_mode() >= 2)) return 0;
    if (c->fine_level == 1) return 0;
    const int k = std::min((c->fine_level == 0 ? c->L + 1 : c->fine_level) - 1, LMAX);
    if ((c->nx >> k) << k != c->nx || (c->ny >> k) << k != c->ny) return 0;
    return k;
}
static void build_coarse(Ctx* c, int k) {
    Ctx::Coarse& m = c->coarse[k];
    if (m.ok) return;
    m.Nc = (uint64_t)(c->nx >> k) * (c->ny >> k);
    m.rp.alloc(c->Ml + 1);
    k_coarse_count<<<blocks_for(c->Ml + 1, 128), 128, 0, c->st>>>(c->Ml, c->rp.p, c->A.p, c->nx, k, m.rp.p);
    check_launch(c, "k_coarse_count");
    exclusive_scan_u64(c, m.rp.p, c->Ml + 1);
    unsigned long long nnz = 0;
    CK(cudaMemcpyAsync(&nnz, m.rp.p + c->Ml, 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    const uint64_t n1 = std::max<unsigned long long>(nnz, 1);
    if (nnz >= (1ull << 32)) throw ConfigError("coarse matrix: more than 2^32 entries");
    m.col.alloc(n1);
    m.val.alloc(n1);
    DBuf<unsigned> kin, kout;
    DBuf<uint2> vin, vout;
    kin.alloc(n1);
    vin.alloc(n1);
    k_coarse_fill<<<blocks_for(c->Ml, 128), 128, 0, c->st>>>(c->Ml, c->rp.p, c->A.p, c->nx, k, m.rp.p, m.col.p,
                                                              m.val.p, kin.p, vin.p);
    check_launch(c, "k_coarse_fill");
    sort_pairs(c, kin, vin, kout, vout, nnz, m.Nc);
    kin.release();
    vin.release();
    m.row.alloc(n1);
    m.valC.alloc(n1);
    if (nnz) {
        k_phiA_gather<<<blocks_for(nnz, 256), 256, 0, c->st>>>(nnz, vout.p, m.val.p, m.row.p, m.valC.p);
        check_launch(c, "k_phiA_gather");
    }
    m.cp.alloc(m.Nc + 1);
    k_bounds<<<blocks_for(m.Nc + 1, 256), 256, 0, c->st>>>(kout.p, nnz, m.Nc, m.cp.p);
    check_launch(c, "k_bounds");
    {   // coarse blocks in 16 x 16 tile order (as build_tile_order)
        std::vector<unsigned> o;
        o.reserve(m.Nc);
        const int T = 16, wx = c->nx >> k, wy = c->ny >> k;
        for (int ty = 0; ty < wy; ty += T)
            for (int tx = 0; tx < wx; tx += T)
                for (int iy = ty; iy < std::min(ty + T, wy); ++iy)
                    for (int ix = tx; ix < std::min(tx + T, wx); ++ix) o.push_back((unsigned)(iy * wx + ix));
        m.order.alloc(m.Nc);
        CK(cudaMemcpyAsync(m.order.p, o.data(), m.Nc * 4, cudaMemcpyHostToDevice, c->st));
    }
    // few, long columns (root phase at cfg4: 4,096 columns of ~3e4 entries, 64 CTAs on 148 SMs:
    // 2.9 ms per launch, profiles/r07/ncu_coarse_root_cfg4.txt): the z-coarse back projection runs
    // over column SEGMENTS and k_g_expand_z adds a column's partials in segment order
    m.seg = c->nzl > 1 ? (m.Nc <= 4096 ? 8 : (m.Nc <= 16384 ? 4 : (m.Nc <= 65536 ? 2 : 1))) : 1;
    if (m.seg > 1) {
        m.cpseg.alloc(m.Nc * m.seg + 1);
        k_seg_bounds<<<blocks_for(m.Nc * m.seg + 1, 256), 256, 0, c->st>>>(m.Nc, m.seg, m.cp.p, m.cpseg.p);
        check_launch(c, "k_seg_bounds");
    }
    CK(cudaStreamSynchronize(c->st));
    c->cub_tmp.release();
    m.nnz = nnz;
    m.ok = true;
}
// 2D: the CSR patch forward and the CSC back projection over Hc
static unsigned fwd2c_launch(Ctx* c, int k) {
    build_coarse(c, k);
    Ctx::Coarse& m = c->coarse[k];
    c->mu_c.ensure(m.Nc);
    if (std::getenv("WAMGPU_COARSE_CHECK") != nullptr) {
        CK(cudaMemsetAsync(c->flag2.p, 0, 4, c->st));
        k_mu_coarse_check<<<blocks_for(c->N, 256), 256, 0, c->st>>>(c->N, c->nx, k, 1, 1, c->mu.p, c->flag2.p);
        int bad = 0;
        CK(cudaMemcpyAsync(&bad, c->flag2.p, 4, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        if (bad) throw NumericError("coarse projection: mu is not constant on the 2^k blocks");
    }
    k_mu_coarse2<<<blocks_for(m.Nc, 256), 256, 0, c->st>>>(m.Nc, c->nx >> k, c->nx, k, c->mu.p, c->mu_c.p);
    check_launch(c, "k_mu_coarse2");
    k_fwd_patch<1, 4, 8, 5, Ent64><<<c->nblk_row, 256, 0, c->st>>>(c->Ml, m.rp.p, Ent64{m.col.p, m.val.p}, c->mu_c.p,
                                                                  c->I0.p, c->d.p, c->q.p, nullptr, c->partial.p,
                                                                  c->flag.p);
    // (counted by forward_fused's check_launch)
    return (unsigned)c->nblk_row;
}
static void back2c_into(Ctx* c, int k, const float* w, double* out) {
    build_coarse(c, k);
    Ctx::Coarse& m = c->coarse[k];
    c->g_c.ensure(m.Nc);
    c->timer_begin(T_BACKC);
    const unsigned nb = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((m.Nc + 7) / 8, (uint64_t)c->sms * 16));
    k_back<0, 12, 1, Ent64><<<nb, 256, 0, c->st>>>(m.Nc, m.cp.p, Ent64{m.row.p, m.valC.p}, w, c->g_c.p, nullptr, nullptr,
                                                   0.0, c->flag.p, -1);
    check_launch(c, "k_back (coarse)");
    k_g_expand2<<<blocks_for(c->N, 256), 256, 0, c->st>>>(c->N, c->nx >> k, c->nx, k, c->g_c.p, out);
    check_launch(c, "k_g_expand2");
    c->timer_end(T_BACKC);
    c->tm.coarse_back_launches++;
    c->tm.proj_updates += (int64_t)m.nnz;
}
// l = Hc mu_c fused with q = I0 exp(-l) and the I-divergence partials; returns the partial count
template <int P>
static unsigned fwd3c_launch_p(Ctx* c, int k, unsigned maxblk) {
    using S = SlabShape<P>;
    Ctx::Coarse& m = c->coarse[k];
    const unsigned nb = std::min<unsigned>(nblk_warp(c, (c->Ml + S::G - 1) / S::G), maxblk);
    k_fwd3s<1, S::LPR, S::SPL, 104, 2, true, P, 8, 2, Ent64><<<nb, 256, 0, c->st>>>(
        c->Ml, 0, c->nzl, m.rp.p, Ent64{m.col.p, m.val.p}, c->mu_c.p, c->I0.p, c->d.p, c->q.p, nullptr,
        c->partial.p, c->flag.p);
    return nb;
}
// z-coarse: l_c = Hc mu_cz on nz / 2^k slices (MODE 0), then q and the I-divergence per slice
template <int PC>
static void fwd3cz_launch_p(Ctx* c, int k, int nzc) {
    using S = SlabShape<PC>;
    Ctx::Coarse& m = c->coarse[k];
    const unsigned nb = nblk_warp(c, (c->Ml + S::G - 1) / S::G);
    k_fwd3s<0, S::LPR, S::SPL, 104, 2, true, PC, 8, 2, Ent64><<<nb, 256, 0, c->st>>>(
        c->Ml, 0, nzc, m.rp.p, Ent64{m.col.p, m.val.p}, c->mu_c.p, nullptr, nullptr, nullptr, c->l_c.p,
        nullptr, c->flag.p);
}
static unsigned fwd3c_launch(Ctx* c, int k, unsigned maxblk) {
    build_coarse(c, k);
    Ctx::Coarse& m = c->coarse[k];
    const int P = slab_stride(c);
    const bool zc = coarse_mode() >= 2;
    const int nzc = c->nzl >> k, Pc = pow2_stride(nzc);
    c->mu_c.ensure(m.Nc * (zc ? Pc : P));
    if (std::getenv("WAMGPU_COARSE_CHECK") != nullptr) {
        sync_mu(c);
        CK(cudaMemsetAsync(c->flag2.p, 0, 4, c->st));
        if (zc)
            k_mu_coarse_check_z<<<blocks_for(c->N * c->nzl, 256), 256, 0, c->st>>>(c->N, c->nx, k, P, c->nzl, c->mu.p, c->flag2.p);
        else
        k_mu_coarse_check<<<blocks_for(c->N * c->nzl, 256), 256, 0, c->st>>>(c->N, c->nx, k, P, c->nzl, c->mu.p, c->flag2.p);
        int bad = 0;
        CK(cudaMemcpyAsync(&bad, c->flag2.p, 4, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        if (bad) throw NumericError("coarse projection: mu is not constant on the 2^k blocks");
    }
    if (zc) {
        c->l_c.ensure(c->Ml * Pc);
        if (c->mu_c_k != k) {   // (the coarse-domain update leaves mu_c ready)
            sync_mu(c);
            k_mu_coarse_z<<<blocks_for(m.Nc * Pc, 256), 256, 0, c->st>>>(m.Nc, c->nx >> k, c->nx, k, P, Pc, nzc,
                                                                         c->mu.p, c->mu_c.p);
            check_launch(c, "k_mu_coarse_z");
        }
        switch (Pc) {
            case 8: fwd3cz_launch_p<8>(c, k, nzc); break;
            case 16: fwd3cz_launch_p<16>(c, k, nzc); break;
            case 32: fwd3cz_launch_p<32>(c, k, nzc); break;
            default: fwd3cz_launch_p<64>(c, k, nzc); break;
        }
        check_launch(c, "k_fwd3s (z-coarse)");
        const unsigned nbz = std::min<unsigned>((unsigned)c->sms * 8, maxblk);
        k_beer_z<<<nbz, 256, 0, c->st>>>(c->Ml, c->nzl, P, Pc, k, c->l_c.p, c->I0.p, c->d.p, c->q.p, c->partial.p,
                                        c->flag.p);
        // (k_beer_z is counted by forward_fused's check_launch)
        return nbz;
    }
    c->mu_c_k = -1;
    k_mu_coarse<<<blocks_for(m.Nc * (P / 4), 256), 256, 0, c->st>>>(m.Nc, c->nx >> k, c->nx, k, P, c->mu.p, c->mu_c.p);
    check_launch(c, "k_mu_coarse");
    unsigned nb = 0;
    switch (P) {
        case 8: nb = fwd3c_launch_p<8>(c, k, maxblk); break;
        case 16: nb = fwd3c_launch_p<16>(c, k, maxblk); break;
        case 32: nb = fwd3c_launch_p<32>(c, k, maxblk); break;
        case 64: nb = fwd3c_launch_p<64>(c, k, maxblk); break;
        default: nb = fwd3c_launch_p<128>(c, k, maxblk); break;
    }
    // (counted by forward_fused's check_launch)
    return nb;
}
// g = expand(Hc^T w): block sums over the coarse CSC, then the block mean on every pixel
template <int P>
static void back3c_launch_p(Ctx* c, int k, const float* w) {
    using S = SlabShape<P>;
    Ctx::Coarse& m = c->coarse[k];
    const unsigned nb = nblk_warp(c, (m.Nc + S::G - 1) / S::G);
    k_back3s<0, S::LPR, S::SPL, 104, 1, false, P, 8, 2, Ent64><<<nb, 256, 0, c->st>>>(
        m.Nc, 0, c->nzl, m.order.p, m.cp.p, Ent64{m.row.p, m.valC.p}, w, c->g_c.p, nullptr, nullptr, 0.0,
        c->flag.p, TileMap{});
}
// WAMGPU_COARSE_DBL=0: z-group sums of q as fp32 (hi, lo) pairs instead of doubles
static bool coarse_dbl() {
    const char* e = std::getenv("WAMGPU_COARSE_DBL");
    return !(e && e[0] == '0');
}
template <int PW>
static void back3cz_launch_p(Ctx* c, int k, int nzw) {
    using S = SlabShape<PW>;
    Ctx::Coarse& m = c->coarse[k];
    const uint64_t ncol = m.Nc * (uint64_t)m.seg;   // seg > 1: column segments in column order (no tile order)
    const unsigned nb = nblk_warp(c, (ncol + S::G - 1) / S::G);
    if constexpr (S::SPL >= 4) {
        if (coarse_dbl()) {   // fp64 z-group sums as the operand: no conversions (default)
            k_back3s<0, S::LPR, S::SPL, 104, 1, true, PW, 8, 2, Ent64, true><<<nb, 256, 0, c->st>>>(
                ncol, 0, nzw, m.seg > 1 ? nullptr : m.order.p, m.seg > 1 ? m.cpseg.p : m.cp.p,
                Ent64{m.row.p, m.valC.p}, c->w_z.p, c->g_c.p, nullptr, nullptr, 0.0, c->flag.p, TileMap{});
            return;
        }
    }
    k_back3s<0, S::LPR, S::SPL, 104, 1, true, PW, 8, 2, Ent64><<<nb, 256, 0, c->st>>>(
        ncol, 0, nzw, m.seg > 1 ? nullptr : m.order.p, m.seg > 1 ? m.cpseg.p : m.cp.p, Ent64{m.row.p, m.valC.p},
        c->w_z.p, c->g_c.p, nullptr, nullptr, 0.0, c->flag.p, TileMap{});
}
static bool coarse_update_on(const Ctx* c) {   // WAMGPU_COARSE_UPDATE=0: full-tile update after expanding g
    const char* e = std::getenv("WAMGPU_COARSE_UPDATE");
    return coarse_mode() >= 2 && c->haar3 && c->nzl > 1 && !(e && e[0] == '0');
}
// expand = false: leave the cube sums in g_c for the coarse-domain update (tile_update_coarse)
static void back3c_into(Ctx* c, int k, const float* w, double* out, bool expand = true) {
    build_coarse(c, k);
    Ctx::Coarse& m = c->coarse[k];
    const int P = slab_stride(c);
    if (coarse_mode() >= 2) {   // z-group sums of w as hi/lo pairs, block x z-group sums of g, cube means
        const int nzc = c->nzl >> k, Pw = pow2_stride(2 * nzc);
        c->w_z.ensure(c->Ml * Pw);
        c->g_c.ensure(m.Nc * m.seg * Pw);
        c->timer_begin(T_BACKC);
        const int dbl = coarse_dbl() && SlabShapeSPL(Pw) >= 4;
        k_qsum_z<<<blocks_for(c->Ml * (Pw / 2), 256), 256, 0, c->st>>>(c->Ml, nzc, P, Pw, k, dbl, w, c->w_z.p);
        check_launch(c, "k_qsum_z");
        switch (Pw) {
            case 8: back3cz_launch_p<8>(c, k, 2 * nzc); break;
            case 16: back3cz_launch_p<16>(c, k, 2 * nzc); break;
            case 32: back3cz_launch_p<32>(c, k, 2 * nzc); break;
            case 64: back3cz_launch_p<64>(c, k, 2 * nzc); break;
            default: back3cz_launch_p<128>(c, k, 2 * nzc); break;
        }
        check_launch(c, "k_back3s (z-coarse)");
        if (expand) {
            k_g_expand_z<<<blocks_for(c->N * c->nzl, 256), 256, 0, c->st>>>(c->N, c->nx >> k, c->nx, k, P, Pw,
                                                                             c->nzl, m.seg, c->g_c.p, out);
            check_launch(c, "k_g_expand_z");
        }
        c->timer_end(T_BACKC);
        c->tm.coarse_back_launches++;
        c->tm.proj_updates += (int64_t)(m.nnz * (uint64_t)(2 * nzc));
        return;
    }
    c->g_c.ensure(m.Nc * P);
    c->timer_begin(T_BACKC);
    switch (P) {
        case 8: back3c_launch_p<8>(c, k, w); break;
        case 16: back3c_launch_p<16>(c, k, w); break;
        case 32: back3c_launch_p<32>(c, k, w); break;
        case 64: back3c_launch_p<64>(c, k, w); break;
        default: back3c_launch_p<128>(c, k, w); break;
    }
    check_launch(c, "k_back3s (coarse)");
    k_g_expand<<<blocks_for(c->N * (P / 2), 256), 256, 0, c->st>>>(c->N, c->nx >> k, c->nx, k, P, c->g_c.p, out);
    check_launch(c, "k_g_expand");
    c->timer_end(T_BACKC);
    c->tm.coarse_back_launches++;
    c->tm.proj_updates += (int64_t)(m.nnz * (uint64_t)c->nzl);
}

// analysis, root solves and synthesis on the (TS >> k)^3 corner of every tile (k_tile3hc):
// beta and the z-coarse mu_c bit-identical to the full-tile update; the pixel mu goes stale
static void tile_update_coarse(Ctx* c, int k) {
    Ctx::Coarse& m = c->coarse[k];
    const int P = slab_stride(c), nzc = c->nzl >> k, Pw = pow2_stride(2 * nzc), Pc = pow2_stride(nzc);
    const int TS = 1 << (c->L - k), T3 = TS * TS * TS;
    c->mu_c.ensure(m.Nc * Pc);
    dim3 grid(c->nx >> c->L, c->ny >> c->L, c->nzl >> c->L);
    const int bs = T3 >= 256 ? 256 : (T3 >= 64 ? 64 : 32);
    const size_t smem = 2ull * T3 * sizeof(double);
    if (smem > 48 * 1024)
        CK(cudaFuncSetAttribute(k_tile3hc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_tile3hc<<<grid, bs, smem, c->st>>>(k, c->nx, c->ny, c->nzl, P, c->L, Pw, m.seg, Pc, c->g_c.p, c->g.p + NV(c),
                                         c->bdata.p, c->act.p, c->off, c->beta.p, c->mu_c.p, c->bp_dbg.p,
                                         c->bm_dbg.p, c->Z0, c->counters.p, c->flag.p);
    check_launch(c, "k_tile3hc");
    c->mu_stale = true;
    c->mu_c_k = k;
    c->stats_k = k;
}

// one wavelet-AM iteration with only the roots active: S = Φ_Aᵀ q̂, root
// solves, ℓ = Φ_A β fused with q̂ and the I-divergence (mu is left stale)
static void phiA_step(Ctx* c) {
    const int wA = c->nx >> c->L, nA = wA * (c->ny >> c->L);
    c->timer_begin(T_PHI);
    const unsigned nbb = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(blocks_for((uint64_t)nA * kPhiSeg * 32, 256),
                                                                              (uint64_t)c->sms * 16));
    k_phiA_back<kPhiSeg><<<nbb, 256, 0, c->st>>>(nA, wA, c->nx, c->phiA_cp.p, c->phiA_row.p, c->phiA_valC.p, c->q.p,
                                                 c->phiA_part.p);
    check_launch(c, "k_phiA_back");
    // view shards: the partials of each (coefficient, segment) over the ranks'
    // own rays are summed (64 KB at cfg2); the update then runs replicated
    if (view_sharded(c)) allreduce_sum(c, c->phiA_part.p, (size_t)nA * kPhiSeg, S_VIEWS);
    k_phiA_update<kPhiSeg><<<blocks_for(nA, 256), 256, 0, c->st>>>(nA, wA, c->nx, c->phiA_part.p, c->bdata.p,
                                                                   c->beta.p, c->Z0, c->bp_dbg.p, c->bm_dbg.p,
                                                                   c->counters.p, c->flag.p);
    check_launch(c, "k_phiA_update");
    const int nparts = (int)std::min<uint64_t>(c->nblk_row, c->partial.n);
    k_phiA_fwd<<<nparts, 256, 0, c->st>>>(c->Ml, c->phiA_rp.p, c->phiA_col.p, c->phiA_val.p, c->beta.p, c->I0.p,
                                          c->d.p, c->q.p, c->partial.p, c->flag.p);
    check_launch(c, "k_phiA_fwd");
    c->timer_end(T_PHI);
    c->tm.phi_launches++;
    k_sum_partials<<<1, 1024, 0, c->st>>>(c->partial.p, nparts, c->scal.p);
    check_launch(c, "k_sum_partials");
    allreduce_sum(c, c->scal.p, 1);
    k_record<<<1, 32, 0, c->st>>>(c->scal.p, c->counters.p, c->objs.p, c->cums.p, c->it.p);
    check_launch(c, "k_record");
    c->mu_stale = true;
}
// separable 3D Haar with only the roots active (kernels_phi.cuh, 3D part)
static void phiA3_step(Ctx* c) {
    const int wA = c->nx >> c->L, nA = wA * (c->ny >> c->L), NK = c->nzl >> c->L, P = slab_stride(c);
    const double cL = cpow3_host(c->L);   // phi(y_s|b,k) = phi_A(y|b) c^L (phi_A carries the in-plane 2^-L)
    const int spl = phiA3_spl(c);
    c->timer_begin(T_PHI);
    const unsigned nbb = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(blocks_for((uint64_t)nA * kPhiSeg * 32, 256),
                                                                              (uint64_t)c->sms * 16));
#define PB(S) k_phiA3_back<kPhiSeg, S><<<nbb, 256, 0, c->st>>>(nA, wA, c->nx, c->nzl, P, c->L, c->phiA_cp.p,       \
                                                               c->phiA_row.p, c->phiA_valC.p, c->q.p, c->phiA_part.p)
    switch (spl) { case 1: PB(1); break; case 2: PB(2); break; default: PB(4); break; }
#undef PB
    check_launch(c, "k_phiA3_back");
    if (view_sharded(c)) allreduce_sum(c, c->phiA_part.p, (size_t)nA * kPhiSeg * NK, S_VIEWS);
    k_phiA3_update<kPhiSeg><<<blocks_for((uint64_t)nA * NK, 256), 256, 0, c->st>>>(
        nA, wA, c->nx, NK, P, c->L, cL, c->phiA_part.p, c->bdata.p, c->beta.p, c->phiA_mblk.p, c->Z0, c->bp_dbg.p,
        c->bm_dbg.p, c->counters.p, c->flag.p);
    check_launch(c, "k_phiA3_update");
    const int nparts = (int)std::min<uint64_t>(nblk_warp(c, c->Ml), c->partial.n);
#define PF(S) k_phiA3_fwd<S><<<nparts, 256, 0, c->st>>>(c->Ml, c->nzl, P, c->L, c->nx, wA, c->phiA_rp.p,          \
                                                        c->phiA_col.p, c->phiA_val.p, c->phiA_mblk.p, c->I0.p, c->d.p, \
                                                        c->q.p, c->partial.p, c->flag.p)
    switch (spl) { case 1: PF(1); break; case 2: PF(2); break; default: PF(4); break; }
#undef PF
    check_launch(c, "k_phiA3_fwd");
    c->timer_end(T_PHI);
    c->tm.phi_launches++;
    k_sum_partials<<<1, 1024, 0, c->st>>>(c->partial.p, nparts, c->scal.p);
    check_launch(c, "k_sum_partials");
    allreduce_sum(c, c->scal.p, 1);
    k_record<<<1, 32, 0, c->st>>>(c->scal.p, c->counters.p, c->objs.p, c->cums.p, c->it.p);
    check_launch(c, "k_record");
    c->mu_stale = true;
    c->bown_stale = true;   // the split update's beta plane is behind the Mallat beta
}
// the split update's own beta plane from the Mallat beta (after root-only iterations)
static void refresh_bown(Ctx* c) {
    if (!c->bown_stale) return;
    c->bown_stale = false;
    if (!wam_split_update(c)) return;
    const TileMap tm = make_tilemap(c);
    k_beta_planes<<<(unsigned)std::min<uint64_t>(blocks_for(tm.CT, 256), (uint64_t)c->sms * 16), 256, 0, c->st>>>(
        tm, slab_stride(c), c->vg, 1, c->bown.p, c->beta.p, c->act.p, c->off, 1);
    check_launch(c, "k_beta_planes");
}

static void sync_mu(Ctx* c) {
    if (!c->mu_stale) return;
    tile_launch(c, 0, nullptr, nullptr);   // mu = Omega beta
    c->mu_stale = false;
}

// separable 3D Haar update split over the view group (kernels3h.cuh): the
// summed chunks [g || b-] of the member's tile rows feed k_tile3h_own, whose
// {mu, beta} planes + counts are all-gathered and unpacked into the mu slab
// (beta stays in the planes until read: sync_beta)
static void tile_update_split(Ctx* c, const TileMap& tm) {
    const int TS = 1 << c->L, P = slab_stride(c);
    const uint64_t CU = u_chunk(tm);
    c->timer_begin(T_UPDATE);
    CK(cudaMemsetAsync(c->ag_send.p + tm.CT, 0, 16, c->st));
    const size_t smem = 2ull * TS * TS * TS * sizeof(double);
    if (smem > 48 * 1024)
        CK(cudaFuncSetAttribute(k_tile3h_own, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_tile3h_own<<<dim3(tm.TX, tm.rows, tm.TZ), 256, smem, c->st>>>(tm, P, c->vg * tm.rows, c->rs_recv.p,
                                                                     c->rs_recv.p + tm.CT, c->bdata.p, c->act.p,
                                                                     c->off, c->ag_send.p, c->bown.p, c->bp_dbg.p,
                                                                     c->bm_dbg.p,
                                                                     c->Z0, c->flag.p);
    check_launch(c, "k_tile3h_own");
    c->timer_end(T_UPDATE);
    all_gather(c, c->ag_send.p, c->ag_recv.p, CU * sizeof(float), S_VIEWS);
    c->timer_begin(T_UPDATE);
    const uint64_t n = tm.CT * c->Rv;
    k_unpack_mu<<<(unsigned)std::min<uint64_t>(blocks_for(n, 256), (uint64_t)c->sms * 16), 256, 0, c->st>>>(
        tm, P, c->Rv, c->ag_recv.p, c->mu.p, c->counters.p);
    check_launch(c, "k_unpack_mu");
    c->timer_end(T_UPDATE);
    c->beta_dirty = true;
}

// slab-Mallat beta from the members' planes (after split updates).  Collective
// over the view group: called at expansions and at the end of every
// iterate/run call, so beta is current at every ABI boundary.
static void sync_beta(Ctx* c) {
    if (!c->beta_dirty) return;
    const TileMap tm = make_tilemap(c);
    all_gather(c, c->bown.p, c->ball.p, tm.CT * sizeof(float), S_VIEWS);
    const uint64_t n = tm.CT * c->Rv;
    k_beta_planes<<<(unsigned)std::min<uint64_t>(blocks_for(n, 256), (uint64_t)c->sms * 16), 256, 0, c->st>>>(
        tm, slab_stride(c), 0, c->Rv, c->ball.p, c->beta.p, c->act.p, c->off, 0);
    check_launch(c, "k_beta_planes");
    c->beta_dirty = false;
}

// split-update buffers at wam_init: T zeroed (b- entries the split never
// writes stay 0), the member's beta plane from the initial beta
static void split_init(Ctx* c) {
    c->beta_dirty = false;
    if (!wam_split_update(c)) return;
    const TileMap tm = make_tilemap(c);
    const uint64_t CU = u_chunk(tm);
    c->rs_send.ensure(2 * tm.CT * c->Rv);
    c->rs_recv.ensure(2 * tm.CT);
    c->ag_send.ensure(CU);
    c->ag_recv.ensure(CU * c->Rv);
    c->bown.ensure(tm.CT);
    c->ball.ensure(tm.CT * c->Rv);
    CK(cudaMemsetAsync(c->rs_send.p, 0, 2 * tm.CT * c->Rv * 8, c->st));
    CK(cudaMemsetAsync(c->ag_send.p, 0, CU * 4, c->st));
    k_beta_planes<<<(unsigned)std::min<uint64_t>(blocks_for(tm.CT, 256), (uint64_t)c->sms * 16), 256, 0, c->st>>>(
        tm, slab_stride(c), c->vg, 1, c->bown.p, c->beta.p, c->act.p, c->off, 1);
    check_launch(c, "k_beta_planes");
}

static void wam_step(Ctx* c) {
    if (c->phiA_ok && c->phiA_L == c->L && phiA_applicable(c) && (c->haar3 ? c->nlist3 == 0 : c->nlist == 0) &&
        !(c->fine_level == 0 && coarse_k(c) > 0)) {
        if (c->haar3) phiA3_step(c);
        else phiA_step(c);
        return;
    }
    refresh_bown(c);
    c->mu_stale = false;   // the update below synthesises mu
    // view-sharded 2D with peer memory: split first (its partial b- rides along
    // as the second half of the fused back projection + all-reduce)
    const bool fused = c->ar.on && c->nz == 1 && !c->haar3;
    const bool split = wam_split_update(c);   // 3D view group: reduce-scatter / own tiles / all-gather
    const TileMap tm = split ? make_tilemap(c) : TileMap{};
    double* bm2 = fused ? c->ar.extra.p : c->g.p + c->N;
    // one GPU, 2D: the signed split (b- over Phi^-) and the back projection
    // (g = H^T q) both read only q and write disjoint halves of [g || b-], so
    // the split runs on the side stream concurrently with the back projection
    // (WAMGPU_SPLIT_OVERLAP=0: sequential)
    static const bool ovl_on = [] {
        const char* e = std::getenv("WAMGPU_SPLIT_OVERLAP");
        return !(e && e[0] == '0');
    }();
    const bool ovl = ovl_on && !c->haar3 && c->nlist && c->nzl == 1 && !fused && !split && !view_sharded(c) &&
                     c->split_variant == 0;
    if (ovl) {
        CK(cudaEventRecord(c->ev_x, c->st));
        CK(cudaStreamWaitEvent(c->st2, c->ev_x, 0));
        c->timer_begin(T_SPLIT, c->st2);
        const unsigned nb = (unsigned)std::min<uint64_t>((c->nlist + 7) / 8, (uint64_t)c->sms * 16);
        k_split<12><<<nb, 256, 0, c->st2>>>(c->nlist, c->list.p, c->cols.p, c->E.p, c->q.p, bm2);
        check_launch(c, "k_split");
        c->timer_end(T_SPLIT, c->st2);
        c->tm.split_launches++;
        c->tm.split_entries += (int64_t)c->nnz_phi;
        CK(cudaEventRecord(c->ev_y, c->st2));
    }
    // block-coarsened projections (kernels3c.cuh) and, in 3D, the update in the coarse domain
    const int ck = (!split && !fused) ? coarse_k(c) : 0;
    const bool cupd = ck > 0 && coarse_update_on(c) && !view_sharded(c);   // (view shards all-reduce the pixel g)
    if (split) {
        back_launch(c, c->q.p, c->rs_send.p, nullptr, true, tm);   // g straight into the tile-major T
        CK(cudaEventRecord(c->ev_x, c->st));
    } else if (!fused) {
        if (ck > 0 && c->nzl == 1) back2c_into(c, ck, c->q.p, c->g.p);
        else if (ck > 0) back3c_into(c, ck, c->q.p, c->g.p, !cupd);
        else back_into(c, c->q.p, c->g.p);
    }
    if (c->haar3 && c->nlist3) {
        c->timer_begin(T_SPLIT);
        const unsigned nb = (unsigned)std::min<uint64_t>((c->nlist3 + 3) / 4, (uint64_t)c->sms * 16);
        double* bm3 = split ? c->rs_send.p + tm.CT * c->Rv : c->g.p + NV(c);   // split: tile-major b- part
#define S3H(S) k_split3h<S><<<nb, 128, 0, c->st>>>(c->nlist3, c->list3.p, c->nx, c->ny, c->nzl, c->np.p, c->E3ray.p, \
                                                   c->E3psi.p, c->q.p, c->act.p, c->off, c->koff, bm3, tm);
#define S3E(S, EE) S3EU(S, EE, 2)
#define S3EU(S, EE, UU)                                                                                            \
    for (int sb_ = 0; sb_ < c->sband_B; ++sb_)                                                                     \
        k_split3h_e<S, EE, UU><<<nb, 128, 0, c->st>>>(c->nlist3, c->list3.p, c->nx, c->ny, c->nzl, c->np.p,        \
                                                      c->E3ray.p, c->E3psi.p, c->q.p, c->act.p, c->off, c->koff,   \
                                                      bm3, tm, c->sband_B > 1 ? c->bptr3.p : nullptr, c->sband_B,  \
                                                      sb_);                                                        \
    launched(c, c->sband_B - 1);
        const int P = slab_stride(c);
        if (c->split_variant == 1 && P >= 32) {
            switch (spl_of(c)) { case 1: S3H(1) break; case 2: S3H(2) break; default: S3H(4) break; }
        } else if (c->split_variant == 2 && P >= 32) {
            switch (P) { case 32: S3E(32, 8) break; case 64: S3E(64, 2) break; default: S3E(128, 2) break; }
        } else if (c->split_variant == 3 && P >= 32) {   // two pipelined rounds of E entries
            switch (P) { case 32: S3E(32, 4) break; case 64: S3E(64, 4) break; default: S3E(128, 2) break; }
        } else if (c->split_variant == 5 && P >= 32) {   // half the entries in flight, half the registers
            switch (P) { case 32: S3EU(32, 4, 1) break; case 64: S3EU(64, 2, 1) break; default: S3EU(128, 1, 1) break; }
        } else if (c->split_variant == 4 && P >= 32) {
            switch (P) { case 32: S3EU(32, 4, 4) break; case 64: S3EU(64, 4, 4) break; default: S3EU(128, 2, 4) break; }
        } else if (c->split_variant == 7) {   // lane per ACTIVE z-block (kernels3h.cuh k_split3z): measured 2x slower
                                              // (cfg3 16.5 vs 7.8, cfg4 92 vs 54 ms per launch, profiles/r06/split3z_ab.txt)
#define S3Z(S) k_split3z<S><<<nb, 128, 0, c->st>>>(c->nlist3, c->list3.p, c->nx, c->ny, c->nzl, c->np.p, c->E3ray.p, \
                                                   c->E3psi.p, c->q.p, c->zbits.p, c->zoff, c->koff, bm3, tm);
            switch (P) {
                case 8: S3Z(8) break;
                case 16: S3Z(16) break;
                case 32: S3Z(32) break;
                case 64: S3Z(64) break;
                default: S3Z(128) break;
            }
#undef S3Z
        } else if ((c->split_variant == 0 || (c->split_variant >= 10 && c->split_variant <= 14 && c->split_variant != 13)) && c->sband_B == 1) {
            // k_split3c (default = 11): cp.async ring of D rounds, dynamic Morton-order scheduling, chunk
            // lane map.  10: 4 warps per block, D 4, 4 CTAs per SM; 11: warp per block; 12: 4 warps per
            // block, 3 CTAs per SM; 14: D 2 (13, D 6, went when the per-entry multipliers took its shared memory).  cfg4 split per run 915 / 889 / 955 / 1073 ms for
            // 10 / 11 / 12 / 13 (k_split3h_e: 1700), cfg3 101 / 98 / 106 / 118 (180): profiles/r07/ab5_split_sectors.txt
#define S3C(Pv, Ev, Dv, Wv, Mv)                                                                                    \
    {                                                                                                              \
        const unsigned nbc = Wv == 1 ? nb : (unsigned)std::min<uint64_t>(c->nlist3, (uint64_t)c->sms * Mv);        \
        CK(cudaMemsetAsync(c->split_ctr.p, 0, 8, c->st));                                                          \
        k_split3c<Pv, Ev, true, Dv, Wv, Mv><<<nbc, 128, 0, c->st>>>(c->nlist3, c->list3.p, c->nx, c->ny, c->nzl,   \
            c->np.p, c->E3ray.p, c->E3psi.p, c->q.p, c->act.p, c->off, c->koff, bm3, tm, c->split_ctr.p);          \
    }
#define S3CV(Pv, Ev)                                                                                               \
    switch (c->split_variant) {                                                                                    \
        case 10: S3C(Pv, Ev, 4, 4, 4) break;                                                                       \
        case 12: S3C(Pv, Ev, 4, 4, 3) break;                                                                       \
        case 14: S3C(Pv, Ev, 2, 4, 4) break;                                                                       \
        default: S3C(Pv, Ev, 4, 1, 4) break;                                                                       \
    }
            switch (P) {   // sharded small slabs: S = 4 slices per lane, the default shape only
                case 8: S3C(8, 16, 3, 1, 4) break;
                case 16: S3C(16, 8, 4, 1, 4) break;
                case 32: S3C(32, 4, 4, 1, 4) break;
                case 64: S3CV(64, 4) break;
                default: S3CV(128, 2) break;
            }
#undef S3CV
#undef S3C
        } else if (c->split_variant == 9 && c->sband_B == 1 && P >= 64) {   // 128-register cap (4 CTAs per SM)
            if (P == 64) k_split3p<64, 4, true, 4><<<nb, 128, 0, c->st>>>(c->nlist3, c->list3.p, c->nx, c->ny, c->nzl, c->np.p,
                                                      c->E3ray.p, c->E3psi.p, c->q.p, c->act.p, c->off, c->koff, bm3, tm);
            else k_split3p<128, 2, true, 4><<<nb, 128, 0, c->st>>>(c->nlist3, c->list3.p, c->nx, c->ny, c->nzl, c->np.p,
                                                      c->E3ray.p, c->E3psi.p, c->q.p, c->act.p, c->off, c->koff, bm3, tm);
        } else if ((c->split_variant == 15 || c->split_variant == 8) && c->sband_B == 1) {
            // 15: k_split3p (per-half q sums, c^l factored out, three-stage register ping-pong pipeline);
            // 8 = the same without the L - Pq form of z-high
#define S3P(S, EE)                                                                                                 \
    if (c->split_variant == 15)                                                                                    \
        k_split3p<S, EE, true><<<nb, 128, 0, c->st>>>(c->nlist3, c->list3.p, c->nx, c->ny, c->nzl, c->np.p,        \
                                                      c->E3ray.p, c->E3psi.p, c->q.p, c->act.p, c->off, c->koff,   \
                                                      bm3, tm);                                                    \
    else                                                                                                           \
        k_split3p<S, EE, false><<<nb, 128, 0, c->st>>>(c->nlist3, c->list3.p, c->nx, c->ny, c->nzl, c->np.p,       \
                                                       c->E3ray.p, c->E3psi.p, c->q.p, c->act.p, c->off, c->koff,  \
                                                       bm3, tm);
            switch (P) {
                case 8: S3P(8, 16) break;
                case 16: S3P(16, 8) break;
                case 32: S3P(32, 4) break;
                case 64: S3P(64, 4) break;
                default: S3P(128, 2) break;
            }
#undef S3P
        } else {   // k_split3h_e (WAMGPU_SPLIT_VARIANT=6, and the ray-banded split): every z-block of a listed block, E entries in flight.
                   // measured: cfg3 (64 slices) E=4 188 ms/run vs 364; cfg4 (128) E=2 1888 vs 2157 (E=4) / 2500;
                   // one pipelined round (U = 1) 182 ms/run at cfg3 vs 188 (U = 2) / 189 (U = 4).
                   // Sharded small slabs: S = P*E/32 = 4 slices per lane.
            switch (P) {
                case 8: S3EU(8, 16, 1) break;
                case 16: S3EU(16, 8, 1) break;
                case 32: S3EU(32, 4, 1) break;
                case 64: S3EU(64, 4, 1) break;
                default: S3EU(128, 2, 1) break;
            }
        }
#undef S3EU
#undef S3E
#undef S3H
        check_launch(c, "k_split3h");
        c->timer_end(T_SPLIT);
        c->tm.split_launches++;
        c->tm.split_entries += (int64_t)c->nnz_phi;
    } else if (!c->haar3 && c->nlist && !ovl) {
        c->timer_begin(T_SPLIT);
        const unsigned nb = (unsigned)std::min<uint64_t>((c->nlist + 7) / 8, (uint64_t)c->sms * 16);
        if (c->nzl == 1) {
            if (c->split_variant == 1)
                k_split<4><<<nb, 256, 0, c->st>>>(c->nlist, c->list.p, c->cols.p, c->E.p, c->q.p, bm2);
            else if (c->split_variant == 2)
                k_split<8><<<nb, 256, 0, c->st>>>(c->nlist, c->list.p, c->cols.p, c->E.p, c->q.p, bm2);
            else if (c->split_variant == 3)
                k_split<16><<<nb, 256, 0, c->st>>>(c->nlist, c->list.p, c->cols.p, c->E.p, c->q.p, bm2);
            else   // measured best at cfg2 (profiles/r01_fwd_patch_sweep.txt)
                k_split<12><<<nb, 256, 0, c->st>>>(c->nlist, c->list.p, c->cols.p, c->E.p, c->q.p, bm2);
        } else {
            double* bm3 = c->g.p + NV(c);
#define S3(S) k_split3<S><<<nb, 256, 0, c->st>>>(c->nlist, c->nzl, slab_stride(c), c->list.p, c->cols.p, c->E.p, \
                                                c->q.p, bm3);
            switch (spl_of(c)) { case 1: S3(1) break; case 2: S3(2) break; default: S3(4) break; }
#undef S3
        }
        check_launch(c, "k_split3");
        c->timer_end(T_SPLIT);
        c->tm.split_launches++;
        c->tm.split_entries += (int64_t)c->nnz_phi;
    }
    if (fused) {
        // inactive details keep b- = 0 (k_tile reads only active ones); the
        // extra half must still be the split's output or zeros
        if (!c->nlist) CK(cudaMemsetAsync(c->ar.extra.p, 0, c->N * 8, c->st));
        back_allreduce(c, c->q.p, c->ar.extra.p);
        CK(cudaMemcpyAsync(c->g.p, c->ar.res.p, 2 * c->N * 8, cudaMemcpyDeviceToDevice, c->st));
    } else if (split) {
        // the g part's reduce-scatter runs on the side stream, overlapping the
        // split (already enqueued on the main stream); the b- part follows it
        CK(cudaStreamWaitEvent(c->st2, c->ev_x, 0));
        reduce_scatter(c, c->rs_send.p, c->rs_recv.p, tm.CT, S_VIEWS, c->st2);
        CK(cudaEventRecord(c->ev_y, c->st2));
        CK(cudaStreamWaitEvent(c->st, c->ev_y, 0));
        reduce_scatter(c, c->rs_send.p + tm.CT * c->Rv, c->rs_recv.p + tm.CT, tm.CT, S_VIEWS, c->st);
        tile_update_split(c, tm);
        c->tm.update_launches++;
        forward_fused(c, true);
        return;
    } else if (view_sharded(c)) {
        allreduce_sum(c, c->g.p, 2 * NV(c), S_VIEWS);   // view shards: partial sums of [g || b-]
    }
    if (ovl) CK(cudaStreamWaitEvent(c->st, c->ev_y, 0));
    c->timer_begin(T_UPDATE);
    if (cupd) {
        tile_update_coarse(c, ck);
    } else {
        tile_launch(c, 1, nullptr, nullptr);
        c->mu_c_k = -1;
        c->stats_k = -1;
    }
    c->timer_end(T_UPDATE);
    c->tm.update_launches++;
    forward_fused(c, true);
}

static void wam_iterate(Ctx* c, int n, wamgpu_record* recs) {
    if (c->algo != 2) throw ContractError("wam: not initialised");
    ensure_records(c, n);
    for (int i = 0; i < n; ++i) {
        wam_step(c);
        CK(cudaEventRecord(c->ev_iter[i], c->st));
        c->iter++;
    }
    sync_beta(c);
    check_flag(c, "wam_iterate");
    fill_records(c, n, recs, c->active);
}

// device tree bytes -> host through a pinned buffer (a pageable 2.4 MB copy
// at cfg3 cost ~1 ms per expansion)
static void act_pinned(Ctx* c) {
    if (c->act_pin_n < c->act_bytes) {
        if (c->act_pin) cudaFreeHost(c->act_pin);
        c->act_pin = nullptr;
        CK(cudaMallocHost(reinterpret_cast<void**>(&c->act_pin), std::max<uint64_t>(c->act_bytes, 1)));
        c->act_pin_n = c->act_bytes;
    }
}
static void act_to_host(Ctx* c, std::vector<uint8_t>& h) {
    act_pinned(c);
    CK(cudaMemcpyAsync(c->act_pin, c->act.p, c->act_bytes, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    std::memcpy(h.data(), c->act_pin, c->act_bytes);
}

// expand_with: blocks of a caller-given tree (e.g. the manifest of another run,
// or the joint tree replayed on one shard) join the criterion's marks; the
// device tree is updated when they add anything
static void merge_add_tree(Ctx* c, std::vector<uint8_t>& h) {
    if (!c->add_tree) return;
    std::atomic<bool> changed{false};
    host_par_chunks(c->act_bytes, 64, [&](uint64_t lo, uint64_t hi, int) {
        bool ch = false;
        for (uint64_t i = lo; i < hi; ++i)
            if (c->add_tree[i] && !h[i]) { h[i] = 1; ch = true; }
        if (ch) changed = true;
    });
    if (changed) {
        act_pinned(c);
        std::memcpy(c->act_pin, h.data(), c->act_bytes);
        CK(cudaMemcpyAsync(c->act.p, c->act_pin, c->act_bytes, cudaMemcpyHostToDevice, c->st));
        CK(cudaStreamSynchronize(c->st));
    }
}

static int64_t wam_expand(Ctx* c, double factor) {
    if (c->algo != 2) throw ContractError("wam: not initialised");
    if (trace_host()) { CK(cudaStreamSynchronize(c->st)); c->t_trace = host_ms(); }
    c->timer_begin(T_EXPAND);
    const bool split = wam_split_update(c);
    TileMap tm;
    if (split) {   // criterion of the member's own tiles from its beta plane
        refresh_bown(c);
        tm = make_tilemap(c);
        const int TS = 1 << c->L;
        const uint64_t ntl = (uint64_t)tm.TX * tm.rows * tm.TZ;
        c->dscratch.ensure(std::max<uint64_t>(ntl, c->act_bytes));
        const size_t smem = 2ull * TS * TS * TS * sizeof(double);
        if (smem > 48 * 1024)
            CK(cudaFuncSetAttribute(k_crit_own, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_crit_own<<<dim3(tm.TX, tm.rows, tm.TZ), 256, smem, c->st>>>(tm, slab_stride(c), c->vg * tm.rows,
                                                                      c->bown.p, c->mu64.p, c->dscratch.p);
        check_launch(c, "k_crit_own");
        k_max_partials<<<1, 256, 0, c->st>>>(c->dscratch.p, ntl, c->scal.p + 1);
        check_launch(c, "k_max_partials");
    } else {
        sync_beta(c);
        tile_launch(c, 0, c->mu64.p, nullptr);     // fp64 criterion image Omega beta (and mu)
        c->mu_stale = false;
    }
    if (c->haar3) {                                 // pin P3: every voxel, no z-sum
        int64_t newly = 0;
        const int nb = 1024;
        if (!split) {
            k_max_slab<<<nb, 256, 0, c->st>>>(c->mu64.p, c->N, c->nzl, slab_stride(c), c->partial.p);
            check_launch(c, "k_max_slab");
            k_max_partials<<<1, 256, 0, c->st>>>(c->partial.p, (uint64_t)nb, c->scal.p + 1);
            check_launch(c, "k_max_partials");
        }
        allreduce_max(c, c->scal.p + 1, 1);
        double mx = 0.0;
        CK(cudaMemcpyAsync(&mx, c->scal.p + 1, 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        if ((mx > 0.0 || c->add_tree) && c->L > 0) {
            std::vector<uint8_t> h(c->act_bytes);
            if (mx > 0.0) {
                CK(cudaMemcpyAsync(c->act_new.p, c->act.p, c->act_bytes, cudaMemcpyDeviceToDevice, c->st));
                uint64_t e0 = 0, e1 = c->N * c->nzl;
                if (split) {   // own tile rows only; the view group merges the marks
                    const uint64_t rowv = (uint64_t)c->nx * c->nzl << c->L;   // voxels per tile row
                    e0 = rowv * (uint64_t)(c->vg * tm.rows);
                    e1 = e0 + rowv * tm.rows;
                }
                k_mark3h<<<blocks_for(e1 - e0, 256), 256, 0, c->st>>>(c->nx, c->ny, c->nzl, slab_stride(c), c->L,
                                                                       c->mu64.p, factor * mx, c->act.p,
                                                                       c->act_new.p, c->off, e0, e1);
                check_launch(c, "k_mark3h");
                c->act.swap(c->act_new);
                if (split) {
                    const unsigned nbk = (unsigned)std::min<uint64_t>(blocks_for(c->act_bytes, 256), c->sms * 16);
                    k_bytes_d<<<nbk, 256, 0, c->st>>>(c->act.p, c->dscratch.p, nullptr, c->act_bytes, 0);
                    check_launch(c, "k_bytes_d");
                    allreduce_max_scope(c, c->dscratch.p, c->act_bytes, S_VIEWS);
                    k_bytes_d<<<nbk, 256, 0, c->st>>>(nullptr, c->dscratch.p, c->act.p, c->act_bytes, 1);
                    check_launch(c, "k_bytes_d");
                }
                act_to_host(c, h);
            } else {
                h = c->act_host;
            }
            merge_add_tree(c, h);
            newly = count_diff(h.data(), c->act_host.data(), c->act_bytes);
            c->act_host.swap(h);
            if (newly > 0) {
                HTRACE("expand3: criterion + mark");
                c->Z0 = compute_z0(c, c->L, false);
                HTRACE("expand3: Z walk + Z0");
                rebuild_psi3(c, c->walk_nlev);
                HTRACE("expand3: Psi rebuild");
                // the tree only grows: 7 details per newly set byte (count_active
                // would rescan all act_bytes on the host: 0.35 ms at cfg3)
                c->active += 7 * newly;
                HTRACE("expand3: count active");
            }
        }
        c->timer_end(T_EXPAND);
        c->tm.expand_events++;
        return newly;
    }
    const double* crit = c->mu64.p;                // nz == 1: the z-sum is the slice
    if (c->nzl > 1 || c->nz > 1) {                 // z-summed image, slabs all-reduced
        c->dscratch.ensure(c->N);
        k_zsum<<<blocks_for(c->N, 256), 256, 0, c->st>>>(c->N, c->nzl, slab_stride(c), c->mu64.p, c->dscratch.p);
        check_launch(c, "k_zsum");
        allreduce_sum(c, c->dscratch.p, c->N, S_SLABS);
        crit = c->dscratch.p;
    }
    const double mx = device_max(c, crit, c->N);
    int64_t newly = 0;
    if ((mx > 0.0 || c->add_tree) && c->L > 0) {
        std::vector<uint8_t> h(c->act_bytes);
        if (mx > 0.0) {
            const double thr = factor * mx;
            CK(cudaMemcpyAsync(c->act_new.p, c->act.p, c->act_bytes, cudaMemcpyDeviceToDevice, c->st));
            k_mark<<<blocks_for(c->N, 256), 256, 0, c->st>>>(c->nx, c->ny, c->L, crit, thr, c->act.p, c->act_new.p,
                                                              c->off);
            check_launch(c, "k_mark");
            c->act.swap(c->act_new);
            act_to_host(c, h);
        } else {
            h = c->act_host;
        }
        merge_add_tree(c, h);
        newly = count_diff(h.data(), c->act_host.data(), c->act_bytes);
        c->act_host.swap(h);
        if (newly > 0) {
            c->fine_level = 0;   // finest level with an active block (coarse projections, kernels3c.cuh)
            for (int l = 1; l <= c->L && !c->fine_level; ++l) {
                const uint8_t* a = c->act_host.data() + c->off.off[l];
                const uint64_t n = (uint64_t)(c->nx >> l) * (c->ny >> l);
                for (uint64_t i = 0; i < n; ++i)
                    if (a[i]) { c->fine_level = l; break; }
            }
            HTRACE("expand: criterion + mark");
            phi_append(c);    // new columns of Phi^-, Z(y) and Z0 of the grown tree
            c->active = count_active(c);
            HTRACE("expand: count active");
        }
    }
    c->timer_end(T_EXPAND);
    c->tm.expand_events++;
    return newly;
}

static void wam_run(Ctx* c, int iters, const int* sched, int nsched, double factor, wamgpu_record* recs) {
    if (c->algo != 2) throw ContractError("wam: not initialised");
    ensure_records(c, iters);
    std::vector<int64_t> act_at(iters);
    int done = 0;
    for (int it = 1; it <= iters; ++it) {
        act_at[it - 1] = c->active;
        wam_step(c);
        CK(cudaEventRecord(c->ev_iter[it - 1], c->st));
        c->iter++;
        ++done;
        for (int k = 0; k < nsched; ++k)
            if (sched[k] == it) { wam_expand(c, factor); break; }
    }
    sync_beta(c);
    check_flag(c, "wam_run");
    if (recs) {
        fill_records(c, iters, recs, 0);
        for (int i = 0; i < iters; ++i) recs[i].active_set = act_at[i];
    }
}

static Ctx* create(int device) {
    auto c = std::make_unique<wamgpu_ctx>();
    c->device = device;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->ev_x, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_y, cudaEventDisableTiming));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) throw CudaError("wamgpu: requires an sm_100a (Blackwell) device");
    c->sms = prop.multiProcessorCount;
    if (const char* e = std::getenv("WAMGPU_FWD_VARIANT")) c->fwd_variant = std::atoi(e);
    if (const char* e = std::getenv("WAMGPU_SPLIT_VARIANT")) c->split_variant = std::atoi(e);
    if (const char* e = std::getenv("WAMGPU_WALK_VARIANT")) c->walk_variant = std::atoi(e);
    if (const char* e = std::getenv("WAMGPU_SLAB_VARIANT")) c->slab_variant = std::atoi(e);
    if (const char* e = std::getenv("WAMGPU_BACK_VARIANT")) c->back_variant = std::atoi(e);
    if (const char* e = std::getenv("WAMGPU_FWD3T")) c->fwd3t_req = std::atoi(e);
    CK(cudaEventCreate(&c->ev_t0));
    CK(cudaEventCreate(&c->ev_a));
    CK(cudaEventCreate(&c->ev_b));
    c->flag.alloc(1);
    c->flag2.alloc(1);
    c->split_ctr.alloc(1);
    c->it.alloc(1);
    c->counters.alloc(2);
    c->scal.alloc(8);
    c->partial.alloc(1024);
    c->t3flag.alloc(1);
    CK(cudaMemsetAsync(c->t3flag.p, 0, 4, c->st));
    CK(cudaMemsetAsync(c->flag.p, 0, 4, c->st));
    CK(cudaMemsetAsync(c->counters.p, 0, 16, c->st));
    CK(cudaStreamSynchronize(c->st));
    return c.release();
}

static void destroy(Ctx* c) {
    cudaSetDevice(c->device);
    // both streams first: the side stream's split may still read A/C/E if an
    // error escaped between its launch and the join in wam_step
    cudaStreamSynchronize(c->st);
    cudaStreamSynchronize(c->st2);
    for (auto& v : c->tev)
        for (auto& p : v) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
    for (auto e : c->ev_iter) cudaEventDestroy(e);
    if (c->ev_t0) cudaEventDestroy(c->ev_t0);
    if (c->ev_a) cudaEventDestroy(c->ev_a);
    if (c->ev_b) cudaEventDestroy(c->ev_b);
    for (void* p : c->ar.opened) cudaIpcCloseMemHandle(p);
    if (c->comm_v) ncclCommDestroy(c->comm_v);
    if (c->comm_z) ncclCommDestroy(c->comm_z);
    if (c->comm) ncclCommDestroy(c->comm);
    c->gstage.release();
    c->lg.reset();
    c->A.release(); c->C.release(); c->E.release();
    for (int k = 0; k < 2; ++k) {
        if (c->pin[k]) cudaFreeHost(c->pin[k]);
        if (c->pin_ev[k]) cudaEventDestroy(c->pin_ev[k]);
    }
    cudaStreamSynchronize(c->st2);
    if (c->act_pin) cudaFreeHost(c->act_pin);
    if (c->ev_x) cudaEventDestroy(c->ev_x);
    if (c->ev_y) cudaEventDestroy(c->ev_y);
    cudaStreamDestroy(c->st2);
    cudaStreamDestroy(c->st);
    delete c;
}

}  // namespace wamgpu

using namespace wamgpu;


#define API_TRY(ctx, ...)                                                             \
    try {                                                                             \
        if (ctx) CK(cudaSetDevice((ctx)->device));                                    \
        __VA_ARGS__;                                                                  \
        return WAMGPU_OK;                                                             \
    } catch (const wamgpu::Error& e) {                                                \
        g_err = e.what();                                                             \
        if (ctx) const_cast<wamgpu_ctx*>(ctx)->err = e.what();     \
        return e.code;                                                                \
    } catch (const std::exception& e) {                                               \
        g_err = e.what();                                                             \
        if (ctx) const_cast<wamgpu_ctx*>(ctx)->err = e.what();     \
        return WAMGPU_ERR_CONTRACT;                                                   \
    }

#define NEED(p) do { if (!(p)) throw ContractError("null argument: " #p); } while (0)

extern "C" {

int wamgpu_version(void) { return 1; }

const char* wamgpu_last_error(const wamgpu_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

int wamgpu_create(int device, wamgpu_ctx** out) {
    const wamgpu_ctx* none = nullptr;
    API_TRY(none, {
        NEED(out);
        *out = create(device);
    })
}

int wamgpu_destroy(wamgpu_ctx* ctx) {
    if (!ctx) return WAMGPU_OK;
    destroy(ctx);
    return WAMGPU_OK;
}

int wamgpu_nccl_unique_id(void* id128) {
    const wamgpu_ctx* none = nullptr;
    API_TRY(none, {
        NEED(id128);
        ncclUniqueId id;
        NK(ncclGetUniqueId(&id));
        std::memcpy(id128, &id, sizeof(id));
    })
}

static void reset_comm(Ctx* c) {
    if (c->comm_v) { ncclCommDestroy(c->comm_v); c->comm_v = nullptr; }
    if (c->comm_z) { ncclCommDestroy(c->comm_z); c->comm_z = nullptr; }
    if (c->comm) { ncclCommDestroy(c->comm); c->comm = nullptr; }
    c->lg.reset();
    c->comm_kind = 0;
    c->rank = 0;
    c->nranks = 1;
}

int wamgpu_set_comm(wamgpu_ctx* ctx, const void* id128, int rank, int nranks) {
    API_TRY(ctx, {
        NEED(ctx);
        if (nranks < 1 || rank < 0 || rank >= nranks) throw ContractError("set_comm: bad rank/nranks");
        if (ctx->have_matrix) throw ContractError("set_comm must precede the system matrix");
        reset_comm(ctx);
        if (id128) {   // nranks == 1 with an id: a 1-rank communicator (exercises the NCCL path)
            ncclUniqueId id;
            std::memcpy(&id, id128, sizeof(id));
            NK(ncclCommInitRank(&ctx->comm, nranks, id, rank));
            ctx->comm_kind = 1;
        } else if (nranks > 1) {
            throw ContractError("set_comm: an ncclUniqueId is required for nranks > 1");
        }
        ctx->rank = rank;
        ctx->nranks = nranks;
    })
}

int wamgpu_set_comm_local(wamgpu_ctx* ctx, int group, int rank, int nranks) {
    API_TRY(ctx, {
        NEED(ctx);
        if (nranks < 1 || rank < 0 || rank >= nranks) throw ContractError("set_comm_local: bad rank/nranks");
        if (ctx->have_matrix) throw ContractError("set_comm_local must precede the system matrix");
        reset_comm(ctx);
        ctx->rank = rank;
        ctx->nranks = nranks;
        if (group < 0) {          // detached shard: this rank's share alone, no exchange
            ctx->comm_kind = nranks > 1 ? 3 : 0;
            return WAMGPU_OK;
        }
        std::shared_ptr<LocalGroup> g;
        {
            std::lock_guard<std::mutex> lk(g_groups_m);
            auto& slot = g_groups[group];
            if (!slot || slot->broken || slot->joined == slot->n) {   // a fresh group under this key
                slot = std::make_shared<LocalGroup>();
                slot->n = nranks;
                slot->stage.assign(nranks, nullptr);
                slot->dev.assign(nranks, -1);
            }
            if (slot->n != nranks) throw ContractError("set_comm_local: nranks differs from the group's");
            if (slot->dev[rank] != -1) throw ContractError("set_comm_local: rank already joined");
            slot->dev[rank] = ctx->device;
            slot->joined++;
            g = slot;
        }
        ctx->lg = g;
        ctx->comm_kind = nranks > 1 ? 2 : 0;
    })
}

int wamgpu_set_partition(wamgpu_ctx* ctx, int view_groups) {
    API_TRY(ctx, {
        NEED(ctx);
        if (ctx->have_matrix) throw ContractError("set_partition must precede the system matrix");
        if (view_groups < 0 || (view_groups > 0 && ctx->nranks % view_groups))
            throw ConfigError("set_partition: view groups must divide the rank count");
        ctx->vgroups_req = view_groups;
    })
}

int wamgpu_debug_guards(uint64_t* checked, uint64_t* bad) {
    const wamgpu_ctx* none = nullptr;
    API_TRY(none, {
        std::string what;
        const auto r = wamgpu::check_guards(&what);
        if (checked) *checked = r.first;
        if (bad) *bad = r.second;
        if (r.second) g_err = what;
    })
}

int wamgpu_set_projector(wamgpu_ctx* ctx, int kind) {
    API_TRY(ctx, {
        NEED(ctx);
        if (kind != 0 && kind != 1) throw ConfigError("set_projector: kind must be 0 (stored matrix) or 1 (on the fly)");
        ctx->fwd3t_req = kind;
        ctx->fwd3t = (kind && ctx->rays_dev.p && ctx->geo_D > 0 && ctx->Ml == (uint64_t)ctx->geo_V * ctx->geo_D) ? 1 : 0;
    })
}
int wamgpu_get_projector(const wamgpu_ctx* ctx, int* state) {
    API_TRY(ctx, {
        NEED(ctx);
        if (state) *state = ctx->fwd3t;
    })
}

int wamgpu_get_partition(const wamgpu_ctx* ctx, int* rv, int* rz, int* s0, int* nzl) {
    API_TRY(ctx, {
        NEED(ctx);
        if (rv) *rv = ctx->Rv;
        if (rz) *rz = ctx->Rz;
        if (s0) *s0 = ctx->s0;
        if (nzl) *nzl = ctx->nzl;
    })
}

// ---- fused back projection + all-reduce over NVLink peer memory ------------
// buffers of this rank: staging R x n, result n, per-tile counters, ready counter
static void ar_alloc(Ctx* c) {
    const int R = c->nranks;
    const uint64_t n = 2 * c->N, ntiles = (n + AR_TILE - 1) / AR_TILE;
    c->ar.n = n;
    c->ar.slot.alloc((uint64_t)R * n);
    c->ar.res.alloc(n);
    c->ar.extra.alloc(c->N);
    c->ar.cnt.alloc(ntiles);
    c->ar.rdy.alloc(1);
    CK(cudaMemsetAsync(c->ar.extra.p, 0, c->N * 8, c->st));
    CK(cudaMemsetAsync(c->ar.cnt.p, 0, ntiles * 8, c->st));
    CK(cudaMemsetAsync(c->ar.rdy.p, 0, 8, c->st));
    CK(cudaStreamSynchronize(c->st));
}

int wamgpu_p2p_export(wamgpu_ctx* ctx, void* blob) {
    API_TRY(ctx, {
        NEED(ctx); NEED(blob);
        Ctx* c = ctx;
        if (c->nranks < 2 || c->nranks > AR_MAX) throw ContractError("p2p: needs 2..8 ranks (set_comm)");
        need_matrix(c);
        if (c->nz != 1) throw ContractError("p2p: the fused all-reduce serves the view-sharded 2D path");
        CK(cudaSetDevice(c->device));
        ar_alloc(c);
        cudaIpcMemHandle_t h[4];
        CK(cudaIpcGetMemHandle(&h[0], c->ar.slot.p));
        CK(cudaIpcGetMemHandle(&h[1], c->ar.res.p));
        CK(cudaIpcGetMemHandle(&h[2], c->ar.cnt.p));
        CK(cudaIpcGetMemHandle(&h[3], c->ar.rdy.p));
        static_assert(sizeof(h) == WAMGPU_P2P_BLOB, "blob size");
        std::memcpy(blob, h, sizeof(h));
    })
}

int wamgpu_p2p_import(wamgpu_ctx* ctx, const void* blobs, int* ok) {
    API_TRY(ctx, {
        NEED(ctx); NEED(blobs);
        Ctx* c = ctx;
        if (!c->ar.slot.p) throw ContractError("p2p_import: p2p_export first");
        CK(cudaSetDevice(c->device));
        // every local failure becomes good = 0; every rank always reaches the
        // agreement all-reduce below (no rank may block in NCCL on another)
        double good = 1.0;
        std::string why;
        try {
            const int R = c->nranks;
            ArArgs a{};
            a.n = c->ar.n;
            a.R = R;
            auto get = [&](int k, int i) {
                cudaIpcMemHandle_t h;
                std::memcpy(&h, (const char*)blobs + (size_t)k * WAMGPU_P2P_BLOB + (size_t)i * sizeof(h), sizeof(h));
                void* p = nullptr;
                CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
                c->ar.opened.push_back(p);
                return p;
            };
            for (int k = 0; k < R; ++k) {
                if (k == c->rank) {
                    a.slot[k] = c->ar.slot.p; a.res[k] = c->ar.res.p; a.cnt[k] = c->ar.cnt.p; a.rdy[k] = c->ar.rdy.p;
                } else {
                    a.slot[k] = (double*)get(k, 0); a.res[k] = (double*)get(k, 1);
                    a.cnt[k] = (unsigned long long*)get(k, 2); a.rdy[k] = (unsigned long long*)get(k, 3);
                }
            }
            c->ar.args = a;
            // self-check (collective, epoch 1): every rank contributes rank+1;
            // a peer that never arrives makes the kernel time out (10 s), not hang
            c->ar.ones.alloc(a.n);
            std::vector<double> v(a.n, (double)(c->rank + 1));
            CK(cudaMemcpyAsync(c->ar.ones.p, v.data(), a.n * 8, cudaMemcpyHostToDevice, c->st));
            ArProdCopy pc{};
            pc.in[c->rank] = c->ar.ones.p;
            ArArgs a1 = a;
            a1.epoch = c->ar.args.epoch = 1;
            a1.r0 = c->rank;
            a1.err = c->flag.p;
            launch_fused_ar(c->sms, c->st, a1, pc, 1);
            check_launch(c, "k_fused_allreduce");
            check_flag(c, "p2p self-check");
            CK(cudaMemcpyAsync(v.data(), c->ar.res.p, a.n * 8, cudaMemcpyDeviceToHost, c->st));
            CK(cudaStreamSynchronize(c->st));
            const double want = 0.5 * R * (R + 1);
            for (double x : v)
                if (x != want) { good = 0.0; why = "wrong self-check sum"; break; }
            c->ar.ones.release();
        } catch (const std::exception& e) {
            good = 0.0;
            why = e.what();
        }
        double* d = nullptr;
        CK(cudaMalloc(&d, 8));
        CK(cudaMemcpyAsync(d, &good, 8, cudaMemcpyHostToDevice, c->st));
        if (c->comm) NK(ncclAllReduce(d, d, 1, ncclDouble, ncclMin, c->comm, c->st));
        CK(cudaMemcpyAsync(&good, d, 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        cudaFree(d);
        c->ar.on = good == 1.0;
        if (ok) *ok = c->ar.on ? 1 : 0;
        if (!c->ar.on && !why.empty()) c->err = "p2p disabled on this rank: " + why;
    })
}

// R logical ranks emulated in ONE cooperative grid on one GPU (B200_PROFILING.md):
// partials R x n -> out R x n (every rank's result)
int wamgpu_selftest_fused_allreduce(int device, int R, uint64_t n, const double* partials, double* out,
                                    int epochs) {
    const wamgpu_ctx* none = nullptr;
    API_TRY(none, {
        NEED(partials); NEED(out);
        if (R < 1 || R > AR_MAX || n == 0 || epochs < 1) throw ContractError("selftest: bad R / n / epochs");
        CK(cudaSetDevice(device));
        int sms = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        cudaStream_t st;
        CK(cudaStreamCreate(&st));
        const uint64_t ntiles = (n + AR_TILE - 1) / AR_TILE;
        std::vector<DBuf<double>> slot(R), res(R), in(R);
        std::vector<DBuf<unsigned long long>> cnt(R), rdy(R);
        DBuf<int> err;
        err.alloc(1);
        CK(cudaMemsetAsync(err.p, 0, 4, st));
        ArArgs a{};
        ArProdCopy pc{};
        a.n = n; a.R = R; a.r0 = 0; a.err = err.p;
        for (int k = 0; k < R; ++k) {
            slot[k].alloc((uint64_t)R * n); res[k].alloc(n); in[k].alloc(n); cnt[k].alloc(ntiles); rdy[k].alloc(1);
            CK(cudaMemsetAsync(cnt[k].p, 0, ntiles * 8, st));
            CK(cudaMemsetAsync(rdy[k].p, 0, 8, st));
            CK(cudaMemcpyAsync(in[k].p, partials + (uint64_t)k * n, n * 8, cudaMemcpyHostToDevice, st));
            a.slot[k] = slot[k].p; a.res[k] = res[k].p; a.cnt[k] = cnt[k].p; a.rdy[k] = rdy[k].p;
            pc.in[k] = in[k].p;
        }
        for (int e = 1; e <= epochs; ++e) {
            a.epoch = (unsigned long long)e;
            for (int k = 0; k < R; ++k) CK(cudaMemsetAsync(res[k].p, 0xff, n * 8, st));   // NaN: must be rewritten
            launch_fused_ar(sms, st, a, pc, R);
            CK(cudaGetLastError());
        }
        for (int k = 0; k < R; ++k) CK(cudaMemcpyAsync(out + (uint64_t)k * n, res[k].p, n * 8, cudaMemcpyDeviceToHost, st));
        int e = 0;
        CK(cudaMemcpyAsync(&e, err.p, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        CK(cudaStreamDestroy(st));
        if (e) throw NumericError("fused all-reduce self-test: a logical rank did not arrive within 10 s");
    })
}

// The production producer (CSC back projection of each rank's own rays + its
// split partial) emulated over R contexts on one GPU: context k plays rank k
// with its own matrix (rows = rank k's shard).  out: R x 2N results.
int wamgpu_selftest_fused_back(wamgpu_ctx* const* ctxs, int R, const double* const* w,
                               const double* const* extra, double* out) {
    const wamgpu_ctx* none = nullptr;
    API_TRY(none, {
        NEED(ctxs); NEED(w); NEED(out);
        if (R < 1 || R > AR_MAX) throw ContractError("selftest: bad R");
        Ctx* c0 = ctxs[0];
        need_matrix(c0);
        CK(cudaSetDevice(c0->device));
        const uint64_t N = c0->N, n = 2 * N, ntiles = (n + AR_TILE - 1) / AR_TILE;
        std::vector<DBuf<double>> slot(R), res(R), ex(R);
        std::vector<DBuf<float>> wf(R);
        std::vector<DBuf<unsigned long long>> cnt(R), rdy(R);
        DBuf<int> err;
        err.alloc(1);
        CK(cudaMemsetAsync(err.p, 0, 4, c0->st));
        ArArgs a{};
        ArProdBack pb{};
        a.n = n; a.R = R; a.r0 = 0; a.epoch = 1; a.err = err.p;
        pb.N = N;
        for (int k = 0; k < R; ++k) {
            Ctx* c = ctxs[k];
            need_matrix(c);
            if (c->N != N || c->device != c0->device) throw ContractError("selftest: contexts must share N and device");
            slot[k].alloc((uint64_t)R * n); res[k].alloc(n); ex[k].alloc(N); cnt[k].alloc(ntiles); rdy[k].alloc(1);
            wf[k].alloc(c->Ml + 1);
            std::vector<float> wv(c->Ml);
            for (uint64_t y = 0; y < c->Ml; ++y) wv[y] = (float)w[k][y];
            CK(cudaMemcpyAsync(wf[k].p, wv.data(), c->Ml * 4, cudaMemcpyHostToDevice, c0->st));
            if (extra && extra[k]) CK(cudaMemcpyAsync(ex[k].p, extra[k], N * 8, cudaMemcpyHostToDevice, c0->st));
            else CK(cudaMemsetAsync(ex[k].p, 0, N * 8, c0->st));
            CK(cudaMemsetAsync(cnt[k].p, 0, ntiles * 8, c0->st));
            CK(cudaMemsetAsync(rdy[k].p, 0, 8, c0->st));
            a.slot[k] = slot[k].p; a.res[k] = res[k].p; a.cnt[k] = cnt[k].p; a.rdy[k] = rdy[k].p;
            pb.cp[k] = c->cp.p; pb.C[k] = c->C.p; pb.w[k] = wf[k].p; pb.extra[k] = ex[k].p;
        }
        launch_fused_ar(c0->sms, c0->st, a, pb, R);
        CK(cudaGetLastError());
        for (int k = 0; k < R; ++k) CK(cudaMemcpyAsync(out + (uint64_t)k * n, res[k].p, n * 8, cudaMemcpyDeviceToHost, c0->st));
        int e = 0;
        CK(cudaMemcpyAsync(&e, err.p, 4, cudaMemcpyDeviceToHost, c0->st));
        CK(cudaStreamSynchronize(c0->st));
        if (e) throw NumericError("fused back + all-reduce self-test: a logical rank did not arrive within 10 s");
    })
}

int wamgpu_set_haar_dim(wamgpu_ctx* ctx, int dim) {
    API_TRY(ctx, {
        NEED(ctx);
        if (dim != 2 && dim != 3) throw ConfigError("haar: dimension must be 2 or 3");
        ctx->haar3 = dim == 3;
        ctx->algo = 0;
    })
}

int wamgpu_set_geometry(wamgpu_ctx* ctx, const wamgpu_geometry* g) {
    API_TRY(ctx, { NEED(ctx); NEED(g); set_geometry(ctx, *g); })
}

int wamgpu_set_grid(wamgpu_ctx* ctx, int nx, int ny, int nz) {
    API_TRY(ctx, {
        NEED(ctx);
        if (nx < 1 || ny < 1 || nz < 1) throw ConfigError("set_grid: invalid grid");
        // the grid shapes everything derived from the matrix (partition, slab
        // stride, tile order, the zA / Phi_A caches): it must come first
        if (ctx->have_matrix) throw ContractError("set_grid: must precede the system matrix");
        ctx->nx = nx; ctx->ny = ny; ctx->nz = nz; ctx->have_grid = true;
    })
}

int wamgpu_set_matrix_csr(wamgpu_ctx* ctx, uint64_t rows, uint64_t cols, uint64_t nnz, const uint64_t* rp,
                          const uint32_t* ci, const double* val) {
    API_TRY(ctx, { NEED(ctx); set_matrix_csr(ctx, rows, cols, nnz, rp, ci, val); })
}

int wamgpu_plan_partition(const wamgpu_geometry* g, int rank, int nranks, int view_groups, int algo, int haar_dim,
                          int levels, wamgpu_plan* out) {
    const wamgpu_ctx* none = nullptr;
    API_TRY(none, {
        NEED(g); NEED(out);
        validate(*g);
        const GridPlan p = make_plan(g->nz, g->views, g->detectors, rank, nranks, view_groups);
        *out = wamgpu_plan{};
        out->view_groups = p.Rv; out->z_groups = p.Rz; out->view_group = p.vg; out->z_group = p.zg;
        out->row_begin = p.row0; out->row_end = p.row1;
        out->slab_begin = p.s0; out->slab_slices = p.nzl;
        int P = 1;
        if (p.nzl > 1) { P = 8; while (P < p.nzl) P *= 2; }
        out->slab_stride = P;
        // the view group's split update (wamgpu.cu am/wam_split_update): its
        // members own disjoint image rows (AM) or rows of 2^L-cube tiles (WAM)
        const bool on = split_update_enabled() && g->nz > 1 && p.Rv > 1;
        if (on && algo == 1 && g->ny % p.Rv == 0) {
            out->split_update = 1;
            out->own_rows = g->ny / p.Rv;
            out->own_row_begin = p.vg * out->own_rows;
        } else if (on && algo == 2 && haar_dim == 3 && levels >= 0 && levels < 20 &&
                   ((g->ny >> levels) % p.Rv) == 0) {
            out->split_update = 1;
            out->own_rows = (g->ny >> levels) / p.Rv;
            out->own_row_begin = p.vg * out->own_rows;
        }
    })
}

int wamgpu_load_matrix_wamh(wamgpu_ctx* ctx, const char* path) {
    API_TRY(ctx, { NEED(ctx); load_matrix_wamh(ctx, path); })
}

int wamgpu_save_matrix_wamh(wamgpu_ctx* ctx, const char* path, int version, int with_csc) {
    API_TRY(ctx, { NEED(ctx); save_matrix_wamh(ctx, path, version, with_csc); })
}

int wamgpu_matrix_info(const wamgpu_ctx* ctx, uint64_t* rows, uint64_t* cols, uint64_t* nnz, uint64_t* r0,
                       uint64_t* r1) {
    API_TRY(ctx, {
        NEED(ctx);
        if (rows) *rows = ctx->M;
        if (cols) *cols = ctx->N;
        if (nnz) *nnz = ctx->nnz;
        if (r0) *r0 = ctx->row0;
        if (r1) *r1 = ctx->row1;
    })
}

int wamgpu_get_matrix_csr(const wamgpu_ctx* ctx, uint64_t* rp, uint32_t* ci, float* val) {
    API_TRY(ctx, {
        NEED(ctx);
        Ctx* c = const_cast<wamgpu_ctx*>(ctx);
        need_matrix(c);
        std::vector<uint2> e(std::max<uint64_t>(c->nnz, 1));
        if (rp) CK(cudaMemcpyAsync(rp, c->rp.p, (c->Ml + 1) * 8, cudaMemcpyDeviceToHost, c->st));
        if (c->nnz) CK(cudaMemcpyAsync(e.data(), c->A.p, c->nnz * 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        for (uint64_t k = 0; k < c->nnz; ++k) {
            if (ci) ci[k] = e[k].x;
            if (val) std::memcpy(val + k, &e[k].y, 4);
        }
    })
}

int wamgpu_get_matrix_csc(const wamgpu_ctx* ctx, uint64_t* cp, uint32_t* ri, float* val) {
    API_TRY(ctx, {
        NEED(ctx);
        Ctx* c = const_cast<wamgpu_ctx*>(ctx);
        need_matrix(c);
        std::vector<uint2> e(std::max<uint64_t>(c->nnz, 1));
        if (cp) CK(cudaMemcpyAsync(cp, c->cp.p, (c->N + 1) * 8, cudaMemcpyDeviceToHost, c->st));
        if (c->nnz) CK(cudaMemcpyAsync(e.data(), c->C.p, c->nnz * 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        for (uint64_t k = 0; k < c->nnz; ++k) {
            if (ri) ri[k] = e[k].x;
            if (val) std::memcpy(val + k, &e[k].y, 4);
        }
    })
}

int wamgpu_forward_project(wamgpu_ctx* ctx, const double* mu, double* l) {
    API_TRY(ctx, {
        NEED(ctx); NEED(mu); NEED(l);
        need_matrix(ctx);
        Ctx* c = ctx;
        c->fscratch.ensure(NV(c));
        c->dscratch.ensure(std::max<uint64_t>(MV(c), 1));
        if (c->nzl == 1) upload_image2(c, mu, c->fscratch.p);
        else upload_slab<float>(c, mu, c->fscratch.p, c->N, c->N, 0);
        forward_plain(c, c->fscratch.p, c->dscratch.p);
        download_slab<double>(c, c->dscratch.p, l, c->Ml, c->Ml, 0, true);
        check_flag(c, "forward_project");
    })
}

int wamgpu_back_project(wamgpu_ctx* ctx, const double* w, double* out) {
    API_TRY(ctx, {
        NEED(ctx); NEED(w); NEED(out);
        need_matrix(ctx);
        Ctx* c = ctx;
        c->fscratch.ensure(std::max<uint64_t>(MV(c), 1));
        c->dscratch.ensure(NV(c));
        upload_slab<float>(c, w, c->fscratch.p, c->Ml, c->Ml, 0, true);
        back_into(c, c->fscratch.p, c->dscratch.p, false);
        if (view_sharded(c)) allreduce_sum(c, c->dscratch.p, NV(c), S_VIEWS);
        download_slab<double>(c, c->dscratch.p, out, c->N, c->N, 0);
    })
}

// predicted_means on caller vectors: q = I0 exp(-l), fp64.
int wamgpu_predicted_means(wamgpu_ctx* ctx, uint64_t n, const double* I0, const double* l, double* q) {
    API_TRY(ctx, {
        NEED(ctx);
        if (n) { NEED(I0); NEED(l); NEED(q); }
        Ctx* c = ctx;
        if (n) {
            DBuf<double> dI, dl, dq;
            DBuf<unsigned long long> bad;
            dI.alloc(n); dl.alloc(n); dq.alloc(n); bad.alloc(1);
            CK(cudaMemcpyAsync(dI.p, I0, n * 8, cudaMemcpyHostToDevice, c->st));
            CK(cudaMemcpyAsync(dl.p, l, n * 8, cudaMemcpyHostToDevice, c->st));
            CK(cudaMemsetAsync(bad.p, 0xff, 8, c->st));
            const int nb = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)c->sms * 8);
            k_pred_means<<<nb, 256, 0, c->st>>>(dI.p, dl.p, dq.p, n, bad.p);
            check_launch(c, "k_pred_means");
            unsigned long long first = 0;
            CK(cudaMemcpyAsync(&first, bad.p, 8, cudaMemcpyDeviceToHost, c->st));
            CK(cudaStreamSynchronize(c->st));
            if (first != ~0ull)
                throw NumericError("predicted_means: non-finite line integral at ray " + std::to_string(first));
            CK(cudaMemcpyAsync(q, dq.p, n * 8, cudaMemcpyDeviceToHost, c->st));
            CK(cudaStreamSynchronize(c->st));
        }
    })
}

// i_divergence on caller vectors: fixed-order fp64 sum.
int wamgpu_i_divergence(wamgpu_ctx* ctx, uint64_t n, const double* d, const double* q, double* out) {
    API_TRY(ctx, {
        NEED(ctx); NEED(out);
        if (n) { NEED(d); NEED(q); }
        Ctx* c = ctx;
        *out = 0.0;
        if (n) {
            const int nb = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)c->sms * 8);
            DBuf<double> dd, dq, part;
            DBuf<unsigned long long> bad;
            dd.alloc(n); dq.alloc(n); part.alloc(nb + 1); bad.alloc(1);
            CK(cudaMemcpyAsync(dd.p, d, n * 8, cudaMemcpyHostToDevice, c->st));
            CK(cudaMemcpyAsync(dq.p, q, n * 8, cudaMemcpyHostToDevice, c->st));
            CK(cudaMemsetAsync(bad.p, 0xff, 8, c->st));
            k_idiv_partials<<<nb, 256, 0, c->st>>>(dd.p, dq.p, n, part.p, bad.p);
            check_launch(c, "k_idiv_partials");
            k_sum_partials<<<1, 1024, 0, c->st>>>(part.p, nb, part.p + nb);
            check_launch(c, "k_sum_partials");
            unsigned long long first = 0;
            CK(cudaMemcpyAsync(&first, bad.p, 8, cudaMemcpyDeviceToHost, c->st));
            CK(cudaMemcpyAsync(out, part.p + nb, 8, cudaMemcpyDeviceToHost, c->st));
            CK(cudaStreamSynchronize(c->st));
            if (first != ~0ull) {
                *out = 0.0;
                throw NumericError("i_divergence: q <= 0 at ray " + std::to_string(first));
            }
        }
    })
}

int wamgpu_set_data(wamgpu_ctx* ctx, const double* d, const double* I0) {
    API_TRY(ctx, {
        NEED(ctx); NEED(d); NEED(I0);
        need_matrix(ctx);
        Ctx* c = ctx;
        std::atomic<int> bad{0};
        host_par(c->Ml, [&](uint64_t lo, uint64_t hi) {
            int b = 0;
            for (int s = 0; s < c->nzl; ++s)
                for (uint64_t y = lo; y < hi; ++y) {
                    const uint64_t id = (uint64_t)(c->s0 + s) * c->M + c->row0 + y;
                    if (!(d[id] >= 0.0)) b |= 1;
                    if (!(I0[id] > 0.0)) b |= 2;
                }
            bad.fetch_or(b);
        });
        if (bad & 1) throw ContractError("TransmissionData: d must be >= 0");
        if (bad & 2) throw ContractError("TransmissionData: I0 must be > 0");
        const uint64_t n = std::max<uint64_t>(MV(c), 1);
        c->d.ensure(n);
        c->I0.ensure(n);
        c->q.ensure(n);
        upload_slab<float>(c, d, c->d.p, c->Ml, c->M, c->row0);
        upload_slab<float>(c, I0, c->I0.p, c->Ml, c->M, c->row0);
        c->have_data = true;
        c->algo = 0;
    })
}

int wamgpu_am_init(wamgpu_ctx* ctx, const double* init_mu) {
    API_TRY(ctx, { NEED(ctx); begin_call(ctx); am_init(ctx, init_mu); end_call(ctx); })
}

int wamgpu_am_iterate(wamgpu_ctx* ctx, int n, wamgpu_record* recs) {
    API_TRY(ctx, {
        NEED(ctx);
        if (n < 0) throw ContractError("iterate: n < 0");
        begin_call(ctx);
        am_iterate(ctx, n, recs);
        end_call(ctx);
    })
}

int wamgpu_wam_init(wamgpu_ctx* ctx, int L, const double* init_beta) {
    API_TRY(ctx, { NEED(ctx); begin_call(ctx); wam_init(ctx, L, init_beta); end_call(ctx); })
}

int wamgpu_wam_iterate(wamgpu_ctx* ctx, int n, wamgpu_record* recs) {
    API_TRY(ctx, {
        NEED(ctx);
        if (n < 0) throw ContractError("iterate: n < 0");
        begin_call(ctx);
        wam_iterate(ctx, n, recs);
        end_call(ctx);
    })
}

int wamgpu_wam_expand(wamgpu_ctx* ctx, double factor, int64_t* newly) {
    API_TRY(ctx, {
        NEED(ctx);
        begin_call(ctx);
        int64_t n = wam_expand(ctx, factor);
        end_call(ctx);
        if (newly) *newly = n;
    })
}

int wamgpu_wam_expand_with(wamgpu_ctx* ctx, double factor, const uint8_t* bits, uint64_t nbytes, int64_t* newly) {
    API_TRY(ctx, {
        NEED(ctx);
        if (ctx->algo != 2) throw ContractError("wam: not initialised");
        if (bits && nbytes != ctx->act_bytes) throw ContractError("expand_with: tree size differs from the state's");
        begin_call(ctx);
        ctx->add_tree = bits;
        int64_t n = 0;
        try {
            n = wam_expand(ctx, factor);
        } catch (...) {
            ctx->add_tree = nullptr;
            throw;
        }
        ctx->add_tree = nullptr;
        end_call(ctx);
        if (newly) *newly = n;
    })
}

int wamgpu_wam_run(wamgpu_ctx* ctx, int iters, const int* sched, int nsched, double factor, wamgpu_record* recs) {
    API_TRY(ctx, {
        NEED(ctx);
        if (iters < 0 || nsched < 0 || (nsched && !sched)) throw ContractError("run: bad schedule");
        for (int k = 1; k < nsched; ++k)
            if (sched[k] < sched[k - 1]) throw ContractError("run: schedule must be sorted");
        begin_call(ctx);
        wam_run(ctx, iters, sched, nsched, factor, recs);
        end_call(ctx);
    })
}

int wamgpu_get_image(const wamgpu_ctx* ctx, double* mu) {
    API_TRY(ctx, {
        NEED(ctx); NEED(mu);
        Ctx* c = const_cast<wamgpu_ctx*>(ctx);
        if (!c->algo) throw ContractError("get_image: no solver state");
        if (c->algo == 2) sync_mu(c);
        if (c->nzl == 1) download_image2(c, c->mu.p, mu);
        else download_slab<float>(c, c->mu.p, mu, c->N, c->N, 0);
    })
}

int wamgpu_get_beta(const wamgpu_ctx* ctx, double* beta) {
    API_TRY(ctx, {
        NEED(ctx); NEED(beta);
        Ctx* c = const_cast<wamgpu_ctx*>(ctx);
        if (c->algo != 2) throw ContractError("get_beta: no wavelet-AM state");
        download_slab<float>(c, c->beta.p, beta, c->N, c->N, 0);
    })
}

int wamgpu_get_q(const wamgpu_ctx* ctx, double* q) {
    API_TRY(ctx, {
        NEED(ctx); NEED(q);
        Ctx* c = const_cast<wamgpu_ctx*>(ctx);
        need_data(c);
        download_slab<float>(c, c->q.p, q, c->Ml, c->Ml, 0, true);
    })
}

int wamgpu_get_tree(const wamgpu_ctx* ctx, uint8_t* bits, uint64_t* nbytes) {
    API_TRY(ctx, {
        NEED(ctx);
        if (bits) std::copy(ctx->act_host.begin(), ctx->act_host.end(), bits);
        if (nbytes) *nbytes = ctx->act_host.size();
    })
}

int wamgpu_get_stats(const wamgpu_ctx* ctx, double* b, double* bp, double* bm) {
    API_TRY(ctx, {
        NEED(ctx);
        Ctx* c = const_cast<wamgpu_ctx*>(ctx);
        if (c->algo != 2) throw ContractError("get_stats: no wavelet-AM state");
        if (c->stats_k > 0 && c->coarse[c->stats_k].ok) {
            // the last update ran in the coarse domain: b+ / b- of the levels below were not
            // produced.  Expand the cube sums still held in g_c and analyse the full tiles.
            const int k = c->stats_k, P = slab_stride(c), nzc = c->nzl >> k, Pw = pow2_stride(2 * nzc);
            k_g_expand_z<<<blocks_for(c->N * c->nzl, 256), 256, 0, c->st>>>(c->N, c->nx >> k, c->nx, k, P, Pw, c->nzl,
                                                                             c->coarse[k].seg, c->g_c.p, c->g.p);
            check_launch(c, "k_g_expand_z");
            tile_launch(c, 3, nullptr, nullptr);
            c->stats_k = -1;
        }
        if (b) download_slab<double>(c, c->bdata.p, b, c->N, c->N, 0);
        if (bp) download_slab<double>(c, c->bp_dbg.p, bp, c->N, c->N, 0);
        if (bm) download_slab<double>(c, c->bm_dbg.p, bm, c->N, c->N, 0);
    })
}

int wamgpu_get_scalars(const wamgpu_ctx* ctx, double* Z0, int64_t* cum, int64_t* degen, int64_t* active) {
    API_TRY(ctx, {
        NEED(ctx);
        Ctx* c = const_cast<wamgpu_ctx*>(ctx);
        unsigned long long cnt[2] = {0, 0};
        CK(cudaMemcpyAsync(cnt, c->counters.p, 16, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
        if (Z0) *Z0 = c->Z0;
        if (cum) *cum = c->algo == 1 ? c->active * c->iter : (int64_t)cnt[0];
        if (degen) *degen = (int64_t)cnt[1];
        if (active) *active = c->active;
    })
}

int wamgpu_get_z_rows(wamgpu_ctx* ctx, double* zrow) {
    API_TRY(ctx, {
        NEED(ctx); NEED(zrow);
        Ctx* c = ctx;
        need_matrix(c);
        if (c->algo == 2 && !c->haar3) {
            if (c->Ml) {
                k_zfix_to_d<<<blocks_for(c->Ml, 256), 256, 0, c->st>>>(c->Ml, c->zfix.p, c->zrow.p);
                check_launch(c, "k_zfix_to_d");
            }
        } else if (c->algo == 2 && c->L > 0) {
            compute_z0(c, c->L, false);
        } else {
            compute_z0(c, c->algo == 2 ? c->L : 0, true);
        }
        CK(cudaMemcpyAsync(zrow, c->zrow.p, c->Ml * 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaStreamSynchronize(c->st));
    })
}

int wamgpu_get_timing(const wamgpu_ctx* ctx, wamgpu_timing* t) {
    API_TRY(ctx, { NEED(ctx); NEED(t); *t = ctx->tm; })
}

int wamgpu_set_kernel_timing(wamgpu_ctx* ctx, int on) {
    API_TRY(ctx, { NEED(ctx); ctx->ktime = on != 0; })
}

int wamgpu_rasterize(const wamgpu_geometry* g, const wamgpu_primitive* prims, int n, double bg, double* mu) {
    const wamgpu_ctx* none = nullptr;
    API_TRY(none, { NEED(g); NEED(mu); if (n && !prims) throw ContractError("null prims"); rasterize(*g, prims, n, bg, mu); })
}

int wamgpu_simulate(const wamgpu_geometry* g, const double* mu, const double* I0, uint64_t seed, int noisy,
                    int threads, double* d) {
    const wamgpu_ctx* none = nullptr;
    API_TRY(none, { NEED(g); NEED(mu); NEED(I0); NEED(d); simulate(*g, mu, I0, seed, noisy != 0, threads, d); })
}

int wamgpu_simulate_device(int device, const wamgpu_geometry* g, const double* mu, const double* I0, uint64_t seed,
                           int noisy, double* d) {
    const wamgpu_ctx* none = nullptr;
    API_TRY(none, {
        NEED(g); NEED(mu); NEED(I0); NEED(d);
        CK(cudaSetDevice(device));
        const std::vector<RayD> rays = ray_table(*g);
        const uint64_t M = rays.size(), N = (uint64_t)g->nx * g->ny, nz = (uint64_t)g->nz;
        std::vector<double> mt(N * nz);   // voxel-major [x][s]: lanes read consecutive slices
        host_par(N, [&](uint64_t lo, uint64_t hi) {
            for (uint64_t x = lo; x < hi; ++x)
                for (uint64_t s = 0; s < nz; ++s) mt[x * nz + s] = mu[s * N + x];
        });
        cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        DBuf<RayDev> dr;
        DBuf<double> dmu, dI0, dd;
        DBuf<int> flag;
        dr.alloc(std::max<uint64_t>(M, 1));
        dmu.alloc(std::max<uint64_t>(N * nz, 1));
        dI0.alloc(std::max<uint64_t>(M * nz, 1));
        dd.alloc(std::max<uint64_t>(M * nz, 1));
        flag.alloc(1);
        CK(cudaMemcpyAsync(dr.p, rays.data(), M * sizeof(RayDev), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(dmu.p, mt.data(), N * nz * 8, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(dI0.p, I0, M * nz * 8, cudaMemcpyHostToDevice, st));
        CK(cudaMemsetAsync(flag.p, 0, 4, st));
        int dev_sms = 148;
        CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, device));
        const unsigned nb = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((M + 7) / 8, (uint64_t)dev_sms * 32));
        if (nz <= 32)
            k_simulate<1><<<nb, 256, 0, st>>>(dr.p, M, g->nx, g->ny, g->nz, g->voxel_size, dmu.p, dI0.p, seed, noisy,
                                              dd.p, flag.p);
        else
            k_simulate<4><<<nb, 256, 0, st>>>(dr.p, M, g->nx, g->ny, g->nz, g->voxel_size, dmu.p, dI0.p, seed, noisy,
                                              dd.p, flag.p);
        CK(cudaGetLastError());
        int f = 0;
        CK(cudaMemcpyAsync(&f, flag.p, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(d, dd.p, M * nz * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        CK(cudaStreamDestroy(st));
        if (f) throw NumericError("simulate: invalid Poisson mean");
    })
}

int wamgpu_host_rays(const wamgpu_geometry* g, double* rays6) {
    const wamgpu_ctx* none = nullptr;
    API_TRY(none, {
        NEED(g); NEED(rays6);
        auto r = ray_table(*g);
        std::memcpy(rays6, r.data(), r.size() * sizeof(RayD));
    })
}

}  // extern "C"
