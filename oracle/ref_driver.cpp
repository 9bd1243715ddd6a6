// ref_driver.cpp — thin C shim over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile with
// -I/root/reference/proj/include into oracle/_ref/libwamref.so (git-ignored,
// shipped to the GPU box as a built artefact).  Nothing here restates the
// reference: every computation is a call into wamrec:: from
// proj/include/wamrec/*.hpp.  It exists to pin the oracle's restatement (and
// the product's device ray tracer) bit-for-bit against the reference:
//   * wamrec::make_parallel_geometry / make_fan_geometry ... geometry.hpp:77-112
//   * wamrec::build_system_matrix ........................... projector.hpp:126-148
//   * wamrec::detail::make_ray / trace_ray .................. projector.hpp:22-119
//   * wamrec::SystemMatrix CSC mirror ....................... system_matrix.hpp:61-75
//   * wamrec::save/load_system_matrix (WAMH cache) .......... system_matrix.hpp:117-158
//   * wamrec::parallel_for .................................. parallel.hpp:22-41
#include <wamrec/errors.hpp>
#include <wamrec/geometry.hpp>
#include <wamrec/image.hpp>
#include <wamrec/parallel.hpp>
#include <wamrec/projector.hpp>
#include <wamrec/system_matrix.hpp>

#include <cstdint>
#include <cstring>
#include <memory>
#include <string>

static thread_local std::string g_err;

static int code_of(const std::exception& e) {
    if (dynamic_cast<const wamrec::ConfigError*>(&e)) return 1;
    if (dynamic_cast<const wamrec::ContractError*>(&e)) return 2;
    if (dynamic_cast<const wamrec::NumericError*>(&e)) return 3;
    if (dynamic_cast<const wamrec::IoError*>(&e)) return 4;
    return 5;
}

#define REF_TRY(...) \
    try { __VA_ARGS__; return 0; } catch (const std::exception& e) { g_err = e.what(); return code_of(e); }

struct ref_matrix {
    wamrec::SystemMatrix m;
};

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// beam 0: make_parallel_geometry, beam 1: make_fan_geometry (flat detector)
int ref_build(int beam, int nx, int ny, int nz, double voxel, int views, int detectors, double spacing,
              double sod, double sdd, ref_matrix** out) {
    REF_TRY({
        wamrec::ScanGeometry g =
            beam == 0 ? wamrec::make_parallel_geometry(nx, ny, nz, voxel, views, detectors, spacing)
                      : wamrec::make_fan_geometry(nx, ny, nz, voxel, views, detectors, spacing, sod, sdd);
        auto r = std::make_unique<ref_matrix>();
        r->m = wamrec::build_system_matrix(g);
        *out = r.release();
    })
}

// Traces an arbitrary ray table (6 doubles per ray) with detail::trace_ray on an
// nx x ny grid: used for the pinned arc detector (P1), whose rays the reference
// cannot construct itself but whose intersection lengths it defines.
int ref_build_from_rays(int nx, int ny, double voxel, uint64_t nrays, const double* rays6, ref_matrix** out) {
    REF_TRY({
        wamrec::ScanGeometry g;
        g.nx = nx; g.ny = ny; g.nz = 1; g.voxel_size = voxel;
        g.detectors = 1; g.detector_spacing = 1.0; g.view_angles = {0.0};
        g.validate();
        std::vector<std::uint64_t> rp{0};
        std::vector<std::uint32_t> ci;
        std::vector<double> val;
        for (uint64_t y = 0; y < nrays; ++y) {
            const double* q = rays6 + 6 * y;
            wamrec::detail::Ray ray{q[0], q[1], q[2], q[3], q[4], q[5]};
            wamrec::detail::trace_ray(g, ray, [&](int ix, int iy, double len) {
                ci.push_back(static_cast<std::uint32_t>(iy) * g.nx + ix);
                val.push_back(len);
            });
            rp.push_back(val.size());
        }
        auto r = std::make_unique<ref_matrix>();
        r->m = wamrec::SystemMatrix(nrays, (std::uint64_t)nx * ny, std::move(rp), std::move(ci), std::move(val));
        *out = r.release();
    })
}

int ref_make_ray(int beam, int nx, int ny, double voxel, int views, int detectors, double spacing, double sod,
                 double sdd, int view, int det, double* ray6) {
    REF_TRY({
        wamrec::ScanGeometry g =
            beam == 0 ? wamrec::make_parallel_geometry(nx, ny, 1, voxel, views, detectors, spacing)
                      : wamrec::make_fan_geometry(nx, ny, 1, voxel, views, detectors, spacing, sod, sdd);
        wamrec::detail::Ray r = wamrec::detail::make_ray(g, view, det);
        ray6[0] = r.ox; ray6[1] = r.oy; ray6[2] = r.dx; ray6[3] = r.dy; ray6[4] = r.tmin; ray6[5] = r.tmax;
    })
}

// trace_ray on a grid WITHOUT validate() (SPEC.md:60-62 examples use 1x1 and 2x2
// grids, which validate() forbids: erratum E3).  Returns entry count.
int ref_trace(int nx, int ny, double voxel, const double* ray6, int cap, int* ix, int* iy, double* len,
              int* count) {
    REF_TRY({
        wamrec::ScanGeometry g;
        g.nx = nx; g.ny = ny; g.voxel_size = voxel;
        wamrec::detail::Ray ray{ray6[0], ray6[1], ray6[2], ray6[3], ray6[4], ray6[5]};
        int n = 0;
        wamrec::detail::trace_ray(g, ray, [&](int a, int b, double l) {
            if (n < cap) { ix[n] = a; iy[n] = b; len[n] = l; }
            ++n;
        });
        *count = n;
    })
}

void ref_free(ref_matrix* m) { delete m; }

int ref_dims(const ref_matrix* r, uint64_t* rows, uint64_t* cols, uint64_t* nnz) {
    REF_TRY({ *rows = r->m.rows(); *cols = r->m.cols(); *nnz = r->m.nnz(); })
}

int ref_csr(const ref_matrix* r, uint64_t* rp, uint32_t* ci, double* val) {
    REF_TRY({
        std::memcpy(rp, r->m.row_ptr().data(), r->m.row_ptr().size() * sizeof(uint64_t));
        std::memcpy(ci, r->m.col_idx().data(), r->m.col_idx().size() * sizeof(uint32_t));
        std::memcpy(val, r->m.values().data(), r->m.values().size() * sizeof(double));
    })
}

int ref_csc(const ref_matrix* r, uint64_t* cp, uint32_t* ri, double* val) {
    REF_TRY({
        std::memcpy(cp, r->m.col_ptr().data(), r->m.col_ptr().size() * sizeof(uint64_t));
        std::memcpy(ri, r->m.row_idx().data(), r->m.row_idx().size() * sizeof(uint32_t));
        std::memcpy(val, r->m.col_values().data(), r->m.col_values().size() * sizeof(double));
    })
}

double ref_row_sum(const ref_matrix* r, uint64_t y) { return r->m.row_sum(y); }

int ref_save(const ref_matrix* r, const char* path) { REF_TRY({ wamrec::save_system_matrix(r->m, path); }) }

int ref_load(const char* path, ref_matrix** out) {
    REF_TRY({
        auto r = std::make_unique<ref_matrix>();
        r->m = wamrec::load_system_matrix(path);
        *out = r.release();
    })
}

int ref_equal(const ref_matrix* a, const ref_matrix* b) { return a->m == b->m ? 1 : 0; }

// Reference host threading primitive: y = H x over CSR rows with
// wamrec::parallel_for (the CPU-baseline threading the SPEC asks for).
int ref_forward(const ref_matrix* r, int threads, const double* mu, double* out) {
    REF_TRY({
        const auto& rp = r->m.row_ptr();
        const auto& ci = r->m.col_idx();
        const auto& v = r->m.values();
        wamrec::parallel_for(r->m.rows(), threads, [&](std::size_t lo, std::size_t hi) {
            for (std::size_t y = lo; y < hi; ++y) {
                double acc = 0.0;
                for (std::uint64_t k = rp[y]; k < rp[y + 1]; ++k) acc += v[k] * mu[ci[k]];
                out[y] = acc;
            }
        });
    })
}

}  // extern "C"
