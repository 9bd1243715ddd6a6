// wamgpu.hpp — header-only C++ host API over the C-ABI of include/wamgpu.h.
//
// It mirrors the reference's reconstruct/iterate interface (SPEC.md:63-98,
// 300-308, 353-389) for C++ callers of the wamrec library.  Functions keep the
// SPEC names and argument meaning; errors are the reference's exception classes
// (proj/include/wamrec/errors.hpp:9-36) re-thrown from the ABI status codes.
// Reference value types are accepted duck-typed (templates), so this header
// does not depend on the reference headers:
//   wamrec::ScanGeometry   (geometry.hpp:21-68)   -> Context::set_geometry
//   wamrec::SystemMatrix   (system_matrix.hpp:20) -> Context::set_matrix
//   wamrec::AttenuationImage (image.hpp:17)       -> mu vectors in its layout
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "wamgpu.h"

// With the reference headers on the include path the ABI status codes are
// re-thrown AS the reference's own classes (wamgpu::ConfigError IS
// wamrec::ConfigError), so a caller's `catch (const wamrec::ConfigError&)`
// keeps working after the switch; without them, look-alike classes stand in.
#if defined(__has_include) && !defined(WAMGPU_NO_WAMREC)
#if __has_include(<wamrec/errors.hpp>)
#include <wamrec/errors.hpp>
#define WAMGPU_HAVE_WAMREC 1
#endif
#endif

namespace wamgpu {

#ifdef WAMGPU_HAVE_WAMREC
using Error = wamrec::Error;                  // errors.hpp:9-13
using ConfigError = wamrec::ConfigError;      // errors.hpp:15-19
using ContractError = wamrec::ContractError;  // errors.hpp:21-25
using NumericError = wamrec::NumericError;    // errors.hpp:27-31
using IoError = wamrec::IoError;              // errors.hpp:33-37
#else
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : Error { using Error::Error; };
struct ContractError : Error { using Error::Error; };
struct NumericError : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };
#endif
struct CudaError : Error { using Error::Error; };   // no reference equivalent

inline void check(int rc, const wamgpu_ctx* c) {
    if (rc == WAMGPU_OK) return;
    const std::string msg = wamgpu_last_error(c);
    switch (rc) {
        case WAMGPU_ERR_CONFIG: throw ConfigError(msg);
        case WAMGPU_ERR_CONTRACT: throw ContractError(msg);
        case WAMGPU_ERR_NUMERIC: throw NumericError(msg);
        case WAMGPU_ERR_IO: throw IoError(msg);
        default: throw CudaError(msg);
    }
}

using Record = wamgpu_record;  // ConvergenceRecord

/// One GPU.  Owns the device-resident system matrix, data and solver state.
class Context {
  public:
    explicit Context(int device = 0) { check(wamgpu_create(device, &c_), nullptr); }
    ~Context() { wamgpu_destroy(c_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    wamgpu_ctx* raw() const { return c_; }

    void set_comm(const void* nccl_id128, int rank, int nranks) { check(wamgpu_set_comm(c_, nccl_id128, rank, nranks), c_); }
    // fused back projection + all-reduce over NVLink peer memory (wamgpu.h):
    // export, all-gather the blobs in rank order, import (collective)
    std::vector<char> p2p_export() {
        std::vector<char> b(WAMGPU_P2P_BLOB);
        check(wamgpu_p2p_export(c_, b.data()), c_);
        return b;
    }
    bool p2p_import(const std::vector<char>& all_blobs) {
        int ok = 0;
        check(wamgpu_p2p_import(c_, all_blobs.data(), &ok), c_);
        return ok != 0;
    }

    /// 3D rank grid: view groups x z-slab groups (after set_comm, before the matrix).
    void set_partition(int view_groups) { check(wamgpu_set_partition(c_, view_groups), c_); }
    /// in-process ranks (one host thread per Context); group < 0: detached shard
    void set_comm_local(int group, int rank, int nranks) { check(wamgpu_set_comm_local(c_, group, rank, nranks), c_); }

    /// build_system_matrix(g) on the device (projector.hpp:126-148).
    void set_geometry(const wamgpu_geometry& g) { check(wamgpu_set_geometry(c_, &g), c_); }

    /// wamrec::ScanGeometry -> device system matrix.
    template <class ScanGeometry>
    void set_scan_geometry(const ScanGeometry& g, bool fan) {
        wamgpu_geometry d{};
        d.nx = g.nx; d.ny = g.ny; d.nz = g.nz; d.voxel_size = g.voxel_size;
        d.detectors = g.detectors; d.detector_spacing = g.detector_spacing;
        d.views = static_cast<int>(g.view_angles.size()); d.view_angles = g.view_angles.data();
        d.beam = fan ? WAMGPU_BEAM_FAN_FLAT : WAMGPU_BEAM_PARALLEL;
        d.source_to_center = g.source_to_center; d.source_to_detector = g.source_to_detector;
        set_geometry(d);
    }

    /// SystemMatrix(rows, cols, row_ptr, col_idx, values) (system_matrix.hpp:24-35).
    template <class SystemMatrix>
    void set_matrix(const SystemMatrix& H, int nx = 0, int ny = 0) {
        if (nx > 0) check(wamgpu_set_grid(c_, nx, ny, 1), c_);
        check(wamgpu_set_matrix_csr(c_, H.rows(), H.cols(), H.nnz(), H.row_ptr().data(), H.col_idx().data(),
                                    H.values().data()), c_);
    }

    /// load_system_matrix(path) (system_matrix.hpp:136-158) straight onto the
    /// device: WAMH v1 (the reference's cache) or v2 (fp32 device layout).
    void load_system_matrix(const std::string& path) { check(wamgpu_load_matrix_wamh(c_, path.c_str()), c_); }
    /// save_system_matrix(m, path) (system_matrix.hpp:117-134); version 2 = fp32
    /// device layout (with_csc: plus the CSC mirror).
    void save_system_matrix(const std::string& path, int version = 1, bool with_csc = false) {
        check(wamgpu_save_matrix_wamh(c_, path.c_str(), version, with_csc ? 1 : 0), c_);
    }

    uint64_t rows() const { uint64_t r = 0; check(wamgpu_matrix_info(c_, &r, nullptr, nullptr, nullptr, nullptr), c_); return r; }
    uint64_t cols() const { uint64_t n = 0; check(wamgpu_matrix_info(c_, nullptr, &n, nullptr, nullptr, nullptr), c_); return n; }

    // ---- core-model
    std::vector<double> forward_project(const std::vector<double>& mu) const {
        std::vector<double> l(local_rows());
        check(wamgpu_forward_project(c_, mu.data(), l.data()), c_);
        return l;
    }
    std::vector<double> back_project(const std::vector<double>& w) const {
        std::vector<double> out(cols());
        check(wamgpu_back_project(c_, w.data(), out.data()), c_);
        return out;
    }
    // SPEC.md:81-98
    std::vector<double> predicted_means(const std::vector<double>& I0, const std::vector<double>& l) const {
        if (I0.size() != l.size()) throw ContractError("predicted_means: length mismatch");
        std::vector<double> q(l.size());
        check(wamgpu_predicted_means(c_, l.size(), I0.data(), l.data(), q.data()), c_);
        return q;
    }
    double i_divergence(const std::vector<double>& d, const std::vector<double>& q) const {
        if (d.size() != q.size()) throw ContractError("i_divergence: length mismatch");
        double v = 0.0;
        check(wamgpu_i_divergence(c_, d.size(), d.data(), q.data(), &v), c_);
        return v;
    }

    // ---- data + solvers
    void set_data(const std::vector<double>& d, const std::vector<double>& I0) {
        if (d.size() != I0.size()) throw ContractError("TransmissionData: d and I0 differ in length");
        check(wamgpu_set_data(c_, d.data(), I0.data()), c_);
    }
    void am_init(const std::vector<double>* init_mu = nullptr) {
        check(wamgpu_am_init(c_, init_mu ? init_mu->data() : nullptr), c_);
    }
    std::vector<Record> am_iterate(int n = 1) {
        std::vector<Record> r(n);
        check(wamgpu_am_iterate(c_, n, r.data()), c_);
        return r;
    }
    void init_state(int levels, const std::vector<double>* init_beta = nullptr) {
        check(wamgpu_wam_init(c_, levels, init_beta ? init_beta->data() : nullptr), c_);
    }
    std::vector<Record> wam_iterate(int n = 1) {
        std::vector<Record> r(n);
        check(wamgpu_wam_iterate(c_, n, r.data()), c_);
        return r;
    }
    int64_t expand_tree(double factor = 0.1) {
        int64_t n = 0;
        check(wamgpu_wam_expand(c_, factor, &n), c_);
        return n;
    }
    /// expand_tree plus the blocks of a given tree (get_tree layout): resume a manifest
    int64_t expand_tree_with(double factor, const std::vector<uint8_t>& tree) {
        int64_t n = 0;
        check(wamgpu_wam_expand_with(c_, factor, tree.data(), tree.size(), &n), c_);
        return n;
    }
    std::vector<Record> run(int iters, const std::vector<int>& schedule, double factor = 0.1) {
        std::vector<Record> r(iters);
        check(wamgpu_wam_run(c_, iters, schedule.data(), static_cast<int>(schedule.size()), factor, r.data()), c_);
        return r;
    }

    // ---- state
    std::vector<double> image() const {
        std::vector<double> mu(cols());
        check(wamgpu_get_image(c_, mu.data()), c_);
        return mu;
    }
    std::vector<double> beta() const {
        std::vector<double> b(cols());
        check(wamgpu_get_beta(c_, b.data()), c_);
        return b;
    }
    std::vector<uint8_t> tree() const {
        uint64_t n = 0;
        check(wamgpu_get_tree(c_, nullptr, &n), c_);
        std::vector<uint8_t> t(n);
        check(wamgpu_get_tree(c_, t.data(), &n), c_);
        return t;
    }
    double Z0() const {
        double z = 0.0;
        check(wamgpu_get_scalars(c_, &z, nullptr, nullptr, nullptr), c_);
        return z;
    }

  private:
    uint64_t local_rows() const {
        uint64_t r0 = 0, r1 = 0;
        check(wamgpu_matrix_info(c_, nullptr, nullptr, nullptr, &r0, &r1), c_);
        return r1 - r0;
    }
    wamgpu_ctx* c_ = nullptr;
};

}  // namespace wamgpu
