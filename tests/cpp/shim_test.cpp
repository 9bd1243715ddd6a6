// shim_test.cpp — the reference's own C++ types driving the B200 path through
// include/wamgpu.hpp (drop-in check).  Built by oracle/Makefile (target shim)
// against the UNMODIFIED reference headers into oracle/_ref/shim_test; run on
// the GPU box by tests/test_gpu_cpp_shim.py.
#include <wamrec/geometry.hpp>
#include <wamrec/projector.hpp>
#include <wamrec/system_matrix.hpp>

#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "wamgpu.hpp"

int main() {
    // reference geometry + reference system matrix (projector.hpp:126)
    wamrec::ScanGeometry g = wamrec::make_fan_geometry(64, 64, 1, 1.0, 90, 128, 1.2, 500.0, 1000.0);
    wamrec::SystemMatrix H = wamrec::build_system_matrix(g);
    wamgpu::Context ctx(0);
    ctx.set_matrix(H, g.nx, g.ny);
    // forward projection vs the reference CSR in f64 (fp32 storage on device)
    std::mt19937_64 rng(7);
    std::uniform_real_distribution<double> U(0.0, 0.05);
    std::vector<double> mu(H.cols());
    for (auto& v : mu) v = (double)(float)U(rng);
    std::vector<double> l = ctx.forward_project(mu);
    double num = 0.0, den = 0.0;
    for (std::uint64_t y = 0; y < H.rows(); ++y) {
        double acc = 0.0;
        for (std::uint64_t k = H.row_ptr()[y]; k < H.row_ptr()[y + 1]; ++k)
            acc += (double)(float)H.values()[k] * mu[H.col_idx()[k]];
        num += (acc - l[y]) * (acc - l[y]);
        den += acc * acc;
    }
    const double rel = std::sqrt(num / den);
    // the same matrix through set_geometry (device Siddon) must be identical
    wamgpu::Context ctx2(0);
    ctx2.set_scan_geometry(g, true);
    std::vector<double> l2 = ctx2.forward_project(mu);
    double diff2 = 0.0;
    for (std::size_t y = 0; y < l.size(); ++y) diff2 = std::max(diff2, std::fabs(l[y] - l2[y]));
    // AM and wavelet AM on noiseless data of a disk
    std::vector<double> mt(H.cols(), 0.0);
    for (int iy = 0; iy < 64; ++iy)
        for (int ix = 0; ix < 64; ++ix)
            if ((ix - 31.5) * (ix - 31.5) + (iy - 31.5) * (iy - 31.5) < 400.0) mt[iy * 64 + ix] = 0.02;
    std::vector<double> I0(H.rows(), 1e5), d(H.rows());
    for (std::uint64_t y = 0; y < H.rows(); ++y) {
        double acc = 0.0;
        for (std::uint64_t k = H.row_ptr()[y]; k < H.row_ptr()[y + 1]; ++k) acc += H.values()[k] * mt[H.col_idx()[k]];
        d[y] = 1e5 * std::exp(-acc);
    }
    ctx.set_data(d, I0);
    ctx.am_init();
    auto ra = ctx.am_iterate(20);
    ctx.init_state(3);
    auto rw = ctx.run(20, {5, 10, 15}, 0.1);
    bool mono = true;
    for (std::size_t i = 1; i < ra.size(); ++i) mono = mono && ra[i].objective <= ra[i - 1].objective * (1 + 1e-6);
    for (std::size_t i = 1; i < rw.size(); ++i) mono = mono && rw[i].objective <= rw[i - 1].objective * (1 + 1e-6);
    bool threw = false;
    try { ctx.init_state(9); } catch (const wamrec::ConfigError&) { threw = true; }   // the reference's class
    // WAMH: the reference's own cache file (save_system_matrix) loads onto the
    // device bit-identical to set_matrix; the device's v1 file loads back
    // through the reference's load_system_matrix as the fp32-rounded matrix
    const std::string ref_file = "/tmp/wamgpu_shim_ref.wamh", dev_file = "/tmp/wamgpu_shim_dev.wamh";
    wamrec::save_system_matrix(H, ref_file);
    wamgpu::Context ctx3(0);
    ctx3.load_system_matrix(ref_file);
    std::vector<double> l3 = ctx3.forward_project(mu);
    double diff3 = 0.0;
    for (std::size_t y = 0; y < l.size(); ++y) diff3 = std::max(diff3, std::fabs(l[y] - l3[y]));
    ctx3.save_system_matrix(dev_file, 1);
    wamrec::SystemMatrix H2 = wamrec::load_system_matrix(dev_file);
    bool wamh = diff3 == 0.0 && H2.rows() == H.rows() && H2.cols() == H.cols() && H2.row_ptr() == H.row_ptr() &&
                H2.col_idx() == H.col_idx();
    for (std::uint64_t k = 0; wamh && k < H.nnz(); ++k) wamh = H2.values()[k] == (double)(float)H.values()[k];
    bool io_threw = false;
    try { ctx3.load_system_matrix("/nonexistent/x.wamh"); } catch (const wamrec::IoError&) { io_threw = true; }
    // standalone core ops: Beer's law on the device line integrals
    // against std::exp, the zero of the I-divergence, and the reference's NumericError
    std::vector<double> qd = ctx.predicted_means(std::vector<double>(l.size(), 1e5), l);
    double qrel = 0.0;
    for (std::size_t y = 0; y < l.size(); ++y) {
        const double e = 1e5 * std::exp(-l[y]);
        qrel = std::max(qrel, std::fabs(qd[y] - e) / e);
    }
    bool core = qrel < 1e-14 && ctx.i_divergence(qd, qd) == 0.0 &&
                std::fabs(ctx.i_divergence({2.0}, {1.0}) - (2.0 * std::log(2.0) - 1.0)) < 1e-15;
    bool num_threw = false;
    try { ctx.i_divergence({1.0, 1.0}, {1.0, 0.0}); } catch (const wamrec::NumericError&) { num_threw = true; }
    core = core && num_threw;
    std::remove(ref_file.c_str());
    std::remove(dev_file.c_str());
    std::printf("forward rel %.3e, set_geometry max diff %.3e, AM obj %.6e -> %.6e, WAM obj %.6e -> %.6e, "
                "active %lld, monotone %d, config error mapped %d, WAMH %d, io error mapped %d, core ops %d (q rel %.1e)\n",
                rel, diff2, ra.front().objective, ra.back().objective, rw.front().objective, rw.back().objective,
                (long long)rw.back().active_set, (int)mono, (int)threw, (int)wamh, (int)io_threw, (int)core, qrel);
    const bool ok = rel < 1e-12 && diff2 == 0.0 && mono && threw && rw.back().objective < rw.front().objective &&
                    wamh && io_threw && core;
    std::printf(ok ? "SHIM OK\n" : "SHIM FAIL\n");
    return ok ? 0 : 1;
}
