// host_model.hpp — host-side helpers of libwamgpu.so (ray table, phantom-sim)
// and the error classes that mirror proj/include/wamrec/errors.hpp:9-36.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/wamgpu.h"

namespace wamgpu {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};
struct ConfigError : Error { explicit ConfigError(const std::string& w) : Error(WAMGPU_ERR_CONFIG, w) {} };
struct ContractError : Error { explicit ContractError(const std::string& w) : Error(WAMGPU_ERR_CONTRACT, w) {} };
struct NumericError : Error { explicit NumericError(const std::string& w) : Error(WAMGPU_ERR_NUMERIC, w) {} };
struct IoError : Error { explicit IoError(const std::string& w) : Error(WAMGPU_ERR_IO, w) {} };
struct CudaError : Error { explicit CudaError(const std::string& w) : Error(WAMGPU_ERR_CUDA, w) {} };

struct RayD { double ox, oy, dx, dy, tmin, tmax; };  // detail::Ray, projector.hpp:16-20

void validate(const wamgpu_geometry& g);
std::vector<double> view_angles(const wamgpu_geometry& g);
std::vector<RayD> ray_table(const wamgpu_geometry& g);
void rasterize(const wamgpu_geometry& g, const wamgpu_primitive* prims, int np, double bg, double* mu);
void simulate(const wamgpu_geometry& g, const double* mu, const double* I0, uint64_t seed, bool noisy,
              int threads, double* d);

}  // namespace wamgpu
