/*
 * wamgpu.h — C-ABI of the B200-native alternating-minimization (AM) iteration
 * of arXiv 1508.04458 (wavelet-domain AM with an adaptive Haar tree, plus the
 * image-domain AM baseline).
 *
 * Drop-in boundary.  The reference exposes C++20 free functions and value
 * types in namespace wamrec (proj/include/wamrec/ and SPEC.md).  Each entry
 * point below replaces one of them; the citation says which.  Conventions
 * (SURVEY.md §8b):
 *   - opaque handle, no exceptions across the ABI; every call returns a status
 *     code mapping 1:1 onto the reference's error classes (errors.hpp:9-36);
 *     wamgpu_last_error(ctx) gives the message (thread-local when ctx == NULL);
 *   - caller-owned HOST arrays are copied in/out and never retained; device
 *     memory is owned by the context;
 *   - calls are synchronous at the ABI; one context is not re-entrant
 *     (iterations are strictly sequential);
 *   - image layout (z*ny + iy)*nx + ix (image.hpp:14), ray layout
 *     z*M_slice + view*detectors + det (projector.hpp:123-125);
 *   - coefficient layout: per-slice Mallat layout of the orthonormal Haar
 *     transform (documented in DESIGN.md §3).
 * Storage on the device is fp32 (h, mu, beta, q, d, I0) with fp64 accumulation
 * of every reduction (north_star; pin P7).
 */
#ifndef WAMGPU_H
#define WAMGPU_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (errors.hpp:9-36) */
#define WAMGPU_OK 0
#define WAMGPU_ERR_CONFIG 1   /* wamrec::ConfigError   errors.hpp:17-20 */
#define WAMGPU_ERR_CONTRACT 2 /* wamrec::ContractError errors.hpp:22-25 */
#define WAMGPU_ERR_NUMERIC 3  /* wamrec::NumericError  errors.hpp:27-30 */
#define WAMGPU_ERR_IO 4       /* wamrec::IoError       errors.hpp:32-35 */
#define WAMGPU_ERR_CUDA 5     /* CUDA / NCCL failure (no reference equivalent) */

#define WAMGPU_BEAM_PARALLEL 0 /* make_parallel_geometry, geometry.hpp:77-92 */
#define WAMGPU_BEAM_FAN_FLAT 1 /* make_fan_geometry,      geometry.hpp:95-112 */
#define WAMGPU_BEAM_FAN_ARC 2  /* equiangular arc detector (pin P1) */

typedef struct wamgpu_ctx wamgpu_ctx;

/* wamrec::ScanGeometry (geometry.hpp:21-68) */
typedef struct {
    int nx, ny, nz;
    double voxel_size;
    int detectors;
    double detector_spacing;  /* beams 0/1 */
    int views;
    const double* view_angles; /* NULL => uniform_angles(views, pi | 2pi), geometry.hpp:70-74 */
    int beam;
    double source_to_center, source_to_detector;
    double fan_angle_step;     /* beam 2 */
} wamgpu_geometry;

/* PhantomSpec primitive */
typedef struct {
    int kind; /* 0 ellipse / ellipsoid, 1 rectangle / box */
    double cx, cy, cz, ax, ay, az, angle, value;
} wamgpu_primitive;

/* ConvergenceRecord */
typedef struct {
    int iter;
    double objective;
    double elapsed_s;
    int64_t active_set;
    int64_t cum_updates;
} wamgpu_record;

/* Per-kernel device timings of the last run (CUDA events on the context stream). */
typedef struct {
    double total_ms;       /* whole run/iterate call, device clock */
    double fwd_ms;         /* sum over launches of the fused forward kernel */
    double back_ms;        /* sum over launches of the back-projection kernel */
    double split_ms;       /* signed-split gather */
    double update_ms;      /* Haar analysis + root solve + synthesis */
    double expand_ms;      /* tree expansion (criterion, Z0, Phi^- rebuild) */
    double comm_ms;        /* NCCL collectives */
    int64_t fwd_launches, back_launches, split_launches, update_launches, expand_events;
    int64_t kernel_launches; /* every kernel of this library launched in the call */
    int64_t split_nnz;       /* Phi^- entries gathered per split launch (last) */
    double phi_ms;           /* iterations over the approximation columns (root-only tree) */
    int64_t phi_launches;    /* such iterations (their back / update / forward are not in the above) */
    double coarse_fwd_ms;    /* forward / back launches over a block-coarsened matrix (wavelet AM while the */
    double coarse_back_ms;   /* finest active tree level is > 1); NOT included in fwd_ms / back_ms */
    int64_t coarse_fwd_launches, coarse_back_launches;
    int64_t proj_updates;    /* ray-voxel updates executed by all forward and back launches above: matrix
                                entries streamed (H or a block-coarsened Hc) x slices processed */
    int64_t split_entries;   /* Phi^- / Psi entries streamed by the split launches above (sum over launches) */
} wamgpu_timing;

int wamgpu_version(void);
const char* wamgpu_last_error(const wamgpu_ctx* ctx);

/* Context on one CUDA device.  Replaces the implicit process-wide state of the
 * reference library (one context per GPU, one process per GPU). */
int wamgpu_create(int device, wamgpu_ctx** out);
int wamgpu_destroy(wamgpu_ctx* ctx);

/* Multi-GPU view sharding (2D): NCCL communicator from a
 * 128-byte ncclUniqueId shared by the caller.  Must precede the matrix. */
int wamgpu_nccl_unique_id(void* id128);
int wamgpu_set_comm(wamgpu_ctx* ctx, const void* id128, int rank, int nranks);
/* In-process ranks: R contexts (any devices, one host thread each) joined
 * under the same group key; collectives are rank-order device reductions
 * between host barriers (bit-identical on every member).  group < 0: a
 * DETACHED shard -- the context computes rank's share of an nranks-way
 * partition alone and skips every exchange (timing one rank's work on one
 * GPU; its results are not a reconstruction).  Must precede the matrix. */
int wamgpu_set_comm_local(wamgpu_ctx* ctx, int group, int rank, int nranks);
/* Rank grid: view_groups Rv x z groups
 * Rz = nranks / Rv, rank = zg*Rv + vg.  2D: views only (Rv = nranks, the
 * default).  Axial 3D: default Rv = 1 (z-slabs, scalars cross GPUs); Rv > 1
 * also splits the views of each slab, whose ranks then sum their partial back
 * projections [H^T q || b-] (fp64) every iteration.  After set_comm, before
 * the matrix. */
int wamgpu_set_partition(wamgpu_ctx* ctx, int view_groups);
int wamgpu_get_partition(const wamgpu_ctx* ctx, int* view_groups, int* z_groups, int* slab_begin,
                         int* slab_slices);

/* Debug (WAMGPU_GUARD=1 in the environment before the first allocation): every
 * device allocation carries 256-byte guard bands and a NaN-filled body; this
 * call checks the bands of all live allocations of the process (checked = how
 * many, bad = how many were overwritten; wamgpu_last_error(NULL) names the
 * first).  Without WAMGPU_GUARD both are 0.  The library's own stand-in for
 * compute-sanitizer memcheck / initcheck where that tool is unavailable. */
int wamgpu_debug_guards(uint64_t* checked, uint64_t* bad);

/* 3D forward projector of an axial stack: kind 0 = slab SpMM over
 * the stored in-plane matrix (projector.hpp:123-148 built once, read per pass);
 * kind 1 = on the fly: every pass re-traces the rays (projector.hpp:52-119 on
 * the device, bit-identical h) and stages the image tiles in shared memory by
 * TMA.  Kind 1 needs a geometry (not an explicit matrix) and >= 17 local
 * slices; the first launch checks that every ray bundle fits its tiles and
 * falls back to kind 0 otherwise.  get: state 0 = stored matrix, 1 = on the fly
 * requested (not launched yet), 2 = on the fly active, -1 = rejected. */
int wamgpu_set_projector(wamgpu_ctx* ctx, int kind);
int wamgpu_get_projector(const wamgpu_ctx* ctx, int* state);

/* The rank grid above, computed on the host without a GPU (the same
 * arithmetic set_geometry applies): rank's view group / z group, its CSR rows
 * [row_begin, row_end) (row = view*detectors + det), its slices
 * [slab_begin, slab_begin + slab_slices) and their slab stride, and, when the
 * view group splits the coefficient update (algo 1 = AM, 2 = WAM; haar_dim,
 * levels of the WAM model), the rows it owns: image rows (AM) or rows of
 * 2^levels-cube tiles (separable-Haar WAM). */
typedef struct {
    int view_groups, z_groups, view_group, z_group;
    uint64_t row_begin, row_end;
    int slab_begin, slab_slices, slab_stride;
    int split_update, own_row_begin, own_rows;
} wamgpu_plan;
int wamgpu_plan_partition(const wamgpu_geometry* g, int rank, int nranks, int view_groups, int algo, int haar_dim,
                          int levels, wamgpu_plan* out);

/* Fused back projection + all-reduce over NVLink peer memory (view-sharded 2D,
 * DESIGN.md §7): replaces the back-projection kernel + ncclAllReduce of
 * [g || b-] by one kernel per rank.  After set_comm and the matrix: every rank
 * exports a WAMGPU_P2P_BLOB-byte blob of CUDA IPC handles, the caller gathers
 * them in rank order (any host transport), and every rank imports the
 * concatenation.  import runs a collective self-check; *ok = 1 when the fused
 * path is active, 0 when the library stays on NCCL. */
#define WAMGPU_P2P_BLOB 256
int wamgpu_p2p_export(wamgpu_ctx* ctx, void* blob);
int wamgpu_p2p_import(wamgpu_ctx* ctx, const void* blobs, int* ok);
/* Test hooks (emulate R ranks in one cooperative grid on one GPU): synthetic
 * partials (R x n -> R x n results), and the production back-projection
 * producer over R contexts holding the R row shards (w[k]: shard k's local rows,
 * extra[k]: N doubles or NULL; out: R x 2N). */
int wamgpu_selftest_fused_allreduce(int device, int R, uint64_t n, const double* partials, double* out,
                                    int epochs);
int wamgpu_selftest_fused_back(wamgpu_ctx* const* ctxs, int R, const double* const* w,
                               const double* const* extra, double* out);

/* System model.  set_geometry replaces build_system_matrix(g)
 * (projector.hpp:126-148): the ray table is built on the host with the
 * reference's make_ray arithmetic (projector.hpp:22-49) and the Siddon traversal
 * (projector.hpp:52-119) runs on the device in fp64; CSR and CSC mirror
 * (system_matrix.hpp:61-75) live in HBM as fp32 values + u32 indices.
 * set_matrix_csr replaces SystemMatrix(rows, cols, row_ptr, col_idx, values)
 * (system_matrix.hpp:24-35): caller's f64 CSR, converted to fp32. */
int wamgpu_set_geometry(wamgpu_ctx* ctx, const wamgpu_geometry* g);
int wamgpu_set_matrix_csr(wamgpu_ctx* ctx, uint64_t rows, uint64_t cols, uint64_t nnz,
                          const uint64_t* row_ptr, const uint32_t* col_idx, const double* values);
/* WAMH system-matrix cache: replaces wamrec::load_system_matrix /
 * save_system_matrix (system_matrix.hpp:87-158).  load reads version 1 (the
 * reference's layout: "WAMH", u32 1, u64 M, N, nnz, row_ptr u64[M+1], col_idx
 * u32[nnz], values f64[nnz]; values converted to fp32 on the way in) or
 * version 2 (this library's device layout: v1 header with version 2, u64 flags
 * (bit 0: CSC present), u32 nx, u32 ny (0 = unknown), row_ptr u64[M+1],
 * {col u32, h f32}[nnz], then with bit 0 col_ptr u64[N+1], {row u32, h f32}[nnz]),
 * streaming only this rank's rows; like set_matrix_csr it must follow
 * set_comm / set_partition / set_grid.  save writes the whole matrix (not from
 * a view shard) as version 1 (f64 values of the fp32 device values) or 2
 * (with_csc: also the CSC mirror).  IoError (4) on open/short read/write
 * failures, bad magic or version, or a size inconsistent with the header. */
int wamgpu_load_matrix_wamh(wamgpu_ctx* ctx, const char* path);
int wamgpu_save_matrix_wamh(wamgpu_ctx* ctx, const char* path, int version, int with_csc);
/* geometry of the image grid for set_matrix_csr users (nx*ny == cols); must
 * precede the matrix (ContractError afterwards: the partition, slab layouts and
 * matrix-derived caches follow the grid) */
int wamgpu_set_grid(wamgpu_ctx* ctx, int nx, int ny, int nz);
int wamgpu_matrix_info(const wamgpu_ctx* ctx, uint64_t* rows, uint64_t* cols, uint64_t* nnz_local,
                       uint64_t* row_begin, uint64_t* row_end);
/* local rows of the device matrix (values as stored, fp32) */
int wamgpu_get_matrix_csr(const wamgpu_ctx* ctx, uint64_t* row_ptr, uint32_t* col_idx, float* values);
int wamgpu_get_matrix_csc(const wamgpu_ctx* ctx, uint64_t* col_ptr, uint32_t* row_idx, float* values);

/* core-model: forward_project(H, mu) and back_project(H, w).
 * mu: N_total doubles; l: local M rows x nz; w: local rows; out: N_total
 * (all-reduced across ranks). */
int wamgpu_forward_project(wamgpu_ctx* ctx, const double* mu, double* l);
int wamgpu_back_project(wamgpu_ctx* ctx, const double* w, double* out);

/* core-model on caller vectors of length n (no matrix needed):
 * predicted_means q(y) = I0(y) exp(-l(y)); a non-finite l(y) -> WAMGPU_ERR_NUMERIC
 * naming the ray.  i_divergence I(d||q) = sum d log(d/q) - d + q with 0 log 0 = 0;
 * any q(y) <= 0 -> WAMGPU_ERR_NUMERIC.  The iteration itself never calls these:
 * its forward kernels fuse both. */
int wamgpu_predicted_means(wamgpu_ctx* ctx, uint64_t n, const double* I0, const double* l, double* q);
int wamgpu_i_divergence(wamgpu_ctx* ctx, uint64_t n, const double* d, const double* q, double* out);

/* TransmissionData: d and I0 over ALL rays (z*M + y); each rank
 * keeps its own view rows. */
int wamgpu_set_data(wamgpu_ctx* ctx, const double* d, const double* I0);

/* am-baseline: init (b = H^T d, Z0 = max row sum, q) and
 * n iterations of mu <- max(0, mu + ln(b^/b)/Z0). */
int wamgpu_am_init(wamgpu_ctx* ctx, const double* init_mu);
int wamgpu_am_iterate(wamgpu_ctx* ctx, int n, wamgpu_record* recs);

/* wavelet model for nz > 1: 2 = per-slice 2D Haar with the z-summed criterion
 * (default), 3 = separable 3D Haar octree with the per-voxel
 * criterion (pin P3, BASELINE cfg3/cfg4).  Takes effect at the next wam_init. */
int wamgpu_set_haar_dim(wamgpu_ctx* ctx, int dim);

/* wavelet-am: init_state, wam_iterate, expand_tree, run. */
int wamgpu_wam_init(wamgpu_ctx* ctx, int levels, const double* init_beta);
int wamgpu_wam_iterate(wamgpu_ctx* ctx, int n, wamgpu_record* recs);
int wamgpu_wam_expand(wamgpu_ctx* ctx, double factor, int64_t* newly_active_blocks);
int wamgpu_wam_run(wamgpu_ctx* ctx, int iters, const int* schedule, int nsched, double factor,
                   wamgpu_record* recs);
/* expand_tree with extra blocks: the union of the criterion's marks and the
 * caller's tree `bits` (layout of wamgpu_get_tree, nbytes = its size; it must
 * satisfy the parent closure, as any tree from get_tree does).  Resumes a tree
 * manifest, or replays another run's tree (factor = +inf: the given blocks
 * only, with the criterion still computed). */
int wamgpu_wam_expand_with(wamgpu_ctx* ctx, double factor, const uint8_t* bits, uint64_t nbytes,
                           int64_t* newly_active_blocks);

/* state read-back */
int wamgpu_get_image(const wamgpu_ctx* ctx, double* mu);   /* AM: mu; WAM: Omega*beta (fp32 storage) */
int wamgpu_get_beta(const wamgpu_ctx* ctx, double* beta);
int wamgpu_get_q(const wamgpu_ctx* ctx, double* q);        /* local rows */
int wamgpu_get_tree(const wamgpu_ctx* ctx, uint8_t* bits, uint64_t* nbytes);
int wamgpu_get_stats(const wamgpu_ctx* ctx, double* b, double* bplus, double* bminus);
int wamgpu_get_scalars(const wamgpu_ctx* ctx, double* Z0, int64_t* cum_updates, int64_t* degenerate,
                       int64_t* active_set);
int wamgpu_get_z_rows(wamgpu_ctx* ctx, double* zrow);      /* per local in-plane ray sum |phi| */
int wamgpu_get_timing(const wamgpu_ctx* ctx, wamgpu_timing* t);
int wamgpu_set_kernel_timing(wamgpu_ctx* ctx, int on);

/* phantom-sim, host-side, f64, seeded counter RNG. */
int wamgpu_rasterize(const wamgpu_geometry* g, const wamgpu_primitive* prims, int nprims, double background,
                     double* mu);
int wamgpu_simulate(const wamgpu_geometry* g, const double* mu_true, const double* I0, uint64_t seed,
                    int noisy, int threads, double* d);
/* the same simulation on a CUDA device: identical
 * trace, sums and counter-based Poisson generator, one warp per ray; the
 * counts equal wamgpu_simulate's (tests/test_gpu_simulate.py). */
int wamgpu_simulate_device(int device, const wamgpu_geometry* g, const double* mu_true, const double* I0,
                           uint64_t seed, int noisy, double* d);
/* the host ray table used by set_geometry (6 doubles per in-plane ray) */
int wamgpu_host_rays(const wamgpu_geometry* g, double* rays6);

#ifdef __cplusplus
}
#endif
#endif
