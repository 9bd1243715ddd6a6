/*
 * wam_oracle.h — C interface of the CPU ORACLE.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load liborc.so.  The
 * product (paper_1508_04458_b200/, libwamgpu.so) never links, loads or calls it.
 *
 * The oracle restates, in plain C++20 on the host, the behaviour of
 *   - the reference headers /root/reference/proj/include/wamrec/ (all headers)
 *     (geometry, make_ray, trace_ray, build_system_matrix, SystemMatrix CSC),
 *   - the SPEC-only operations of SPEC.md (core-model, phantom-sim,
 *     haar-multires, am-baseline, wavelet-am) and PAPER.md Algorithm 1.
 * See wam_oracle.cpp for per-function file:line citations.
 */
#ifndef WAM_ORACLE_H
#define WAM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: same numbering as include/wamgpu.h (errors.hpp:9-36) */
enum { ORC_OK = 0, ORC_ERR_CONFIG = 1, ORC_ERR_CONTRACT = 2, ORC_ERR_NUMERIC = 3, ORC_ERR_IO = 4 };

/* beam: 0 parallel (geometry.hpp:77-92), 1 fan flat detector (geometry.hpp:95-112),
 *       2 fan equiangular arc detector (pin P1) */
typedef struct {
    int nx, ny, nz;
    double voxel_size;
    int detectors;
    double detector_spacing;   /* beam 0/1: detector pitch; beam 2: unused */
    int views;
    const double* view_angles; /* NULL => uniform_angles(views, pi or 2pi) */
    int beam;
    double source_to_center, source_to_detector;
    double fan_angle_step;     /* beam 2: delta-gamma (radians) */
} orc_geometry;

typedef struct {
    int kind;                  /* 0 ellipse(oid), 1 rectangle(box) */
    double cx, cy, cz, ax, ay, az, angle, value;
} orc_primitive;

typedef struct {
    int iter;
    double objective;
    double elapsed_s;
    int64_t active_set;
    int64_t cum_updates;
} orc_record;

typedef struct orc_problem orc_problem;

const char* orc_last_error(void);

/* mirror = 0: reference-faithful f64 storage (image.hpp:54, system_matrix.hpp:80)
 * mirror = 1: fp32 storage + fp64 accumulation, mirroring the GPU (pin P7) */
int orc_create(const orc_geometry* g, int mirror, int threads, orc_problem** out);
/* flags: ORC_SLIM = CSR only (no exact-h copy, no CSC; fp32 h in mirror mode):
 * the memory mode for cfg4 (1.87e9 entries per slice).  Results are
 * bit-identical to the full problem's (back projection by an ascending-ray
 * CSR scatter, the CSC's order); get_csr values / get_csc are unavailable. */
#define ORC_SLIM 1
int orc_create_ex(const orc_geometry* g, int mirror, int threads, int flags, orc_problem** out);
/* explicit-H problem (SPEC.md:70, 79, 307 examples): CSR over an nx*ny grid */
int orc_create_csr(uint64_t M, int nx, int ny, const uint64_t* row_ptr, const uint32_t* col,
                   const double* val, int mirror, int threads, orc_problem** out);
void orc_destroy(orc_problem* p);
int orc_dims(const orc_problem* p, uint64_t* M_slice, uint64_t* N_slice, uint64_t* nnz, int* nz);
/* CSR as built (f64 values, exactly what build_system_matrix returns) */
int orc_get_csr(const orc_problem* p, uint64_t* row_ptr, uint32_t* col, double* val);
int orc_get_csc(const orc_problem* p, uint64_t* col_ptr, uint32_t* row, double* val);
/* ray table (ox, oy, dx, dy, tmin, tmax) per in-plane ray */
int orc_get_rays(const orc_problem* p, double* rays6);

/* core-model; vectors span all nz slices */
int orc_forward_project(const orc_problem* p, const double* mu, double* out);
int orc_back_project(const orc_problem* p, const double* w, double* out);
int orc_predicted_means(uint64_t n, const double* I0, const double* l, double* q);
int orc_i_divergence(uint64_t n, const double* d, const double* q, double* out);

/* phantom-sim */
int orc_rasterize(const orc_geometry* g, const orc_primitive* prims, int nprims,
                  double background, double* mu_out);
int orc_simulate(const orc_problem* p, const double* mu_true, const double* I0,
                 uint64_t seed, int noisy, double* d_out);
double orc_uniform(uint64_t seed, uint64_t stream, uint64_t k);
double orc_poisson(uint64_t seed, uint64_t stream, double mean);

/* haar-multires, Mallat layout per slice */
int orc_dwt2(int nx, int ny, int nslices, int L, const double* in, double* out);
int orc_idwt2(int nx, int ny, int nslices, int L, const double* in, double* out);

/* separable 3D Haar (pin P3): volume z-major, 3D Mallat layout */
int orc_dwt3(int nx, int ny, int nz, int L, const double* in, double* out);
int orc_idwt3(int nx, int ny, int nz, int L, const double* in, double* out);
/* wavelet model: 2 = per-slice 2D Haar, 3 = separable 3D Haar (pin P3) */
int orc_set_haar_dim(orc_problem* p, int dim);

/* root solver (errata E1/E2); returns 0 updated, 1 skipped, 2 degenerate */
int orc_solve_update(double b, double bp, double bm, double Z0, double beta, double* out);

/* am-baseline */
int orc_am_init(orc_problem* p, const double* d, const double* I0, const double* init_mu);
int orc_am_iterate(orc_problem* p, int n, orc_record* recs);
/* clamp = 0 disables the max(0, .) of SPEC.md:317 (reduction-property test) */
int orc_am_set_clamp(orc_problem* p, int clamp);
int orc_am_get(const orc_problem* p, double* mu, double* q, double* Z0, double* bdata);

/* wavelet-am */
int orc_wam_init(orc_problem* p, const double* d, const double* I0, int L,
                 const double* init_beta);
int orc_wam_iterate(orc_problem* p, int n, orc_record* recs);
int orc_wam_expand(orc_problem* p, double factor, int64_t* newly_active);
int orc_wam_run(orc_problem* p, int iters, const int* schedule, int nsched, double factor,
                orc_record* recs);
int orc_wam_get(const orc_problem* p, double* beta, double* mu, double* q, double* Z0);
/* tree bitmaps: level l = 1..L concatenated, (ny>>l)*(nx>>l) bytes each */
int orc_wam_tree(const orc_problem* p, uint8_t* bits, uint64_t* nbytes);
/* per-z (Mallat index, slice 0) surrogate stats of the last iteration */
int orc_wam_stats(const orc_problem* p, double* b, double* bp, double* bm);
int orc_wam_counters(const orc_problem* p, int64_t* cum_updates, int64_t* degenerate,
                     int64_t* active_set);
/* Z0 of the current tree computed from scratch (per-ray |phi| sums, Eq. 1.61) */
int orc_wam_z0_rows(const orc_problem* p, double* zrow);
/* explicit phi column of Mallat coefficient z (slice 0): returns nnz, fills rows/vals */
int orc_phi_column(const orc_problem* p, int L, uint32_t z, uint32_t* rows, double* vals,
                   uint64_t cap, uint64_t* nnz);

#ifdef __cplusplus
}
#endif
#endif
