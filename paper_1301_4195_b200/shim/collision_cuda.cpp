// collision_cuda.hpp over the C ABI (include/boltz_cuda.h); see the header.
#include "collision_cuda.hpp"

#include <string>

#include "boltz/errors.hpp"

namespace boltz {
namespace {

[[noreturn]] void throw_gpu(int rc, const char* where) {
    const std::string m = std::string(where) + ": " + boltz_last_error();
    switch (rc) {
        case BOLTZ_ERR_CONFIG: throw ConfigError(m);
        case BOLTZ_ERR_IO: throw IoError(m);
        case BOLTZ_ERR_NUMERIC: throw NumericError(m);
        default: throw Error(static_cast<ErrorCategory>(rc), "CUDA: " + m);
    }
}

void gpu_check(int rc, const char* where) {
    if (rc != BOLTZ_OK) throw_gpu(rc, where);
}

double r0_of(const VelocityGrid& g, const GpuKernelSpec& k) { return k.r0 > 0.0 ? k.r0 : g.half_width; }

}  // namespace

CollisionGpu::CollisionGpu(const VelocityGrid& grid, const GpuKernelSpec& k, std::span<const double> G, int device)
    : grid_(grid) {
    const std::size_t n3 = grid.size();
    if (G.size() != n3 * n3) throw ConfigError("CollisionGpu: weight table must hold N^6 values");
    gpu_check(boltz_create(grid.n, grid.half_width, k.lambda, k.beta, r0_of(grid, k), G.data(), device, &ctx_),
              "CollisionGpu");
    // the reference passes one cell per call: K2 schedule by batch size
    gpu_check(boltz_set_schedule(ctx_, 6), "CollisionGpu");
}

CollisionGpu::CollisionGpu(const VelocityGrid& grid, const GpuKernelSpec& k, int device) : grid_(grid) {
    gpu_check(boltz_create_generated(grid.n, grid.half_width, k.lambda, k.beta, r0_of(grid, k), 64, device, &ctx_),
              "CollisionGpu");
    gpu_check(boltz_set_schedule(ctx_, 6), "CollisionGpu");
}

CollisionGpu::~CollisionGpu() { boltz_destroy(ctx_); }

int64_t CollisionGpu::cells(std::size_t values) const {
    if (values == 0 || values % grid_.size()) throw ConfigError("span is not a whole number of N^3 cells");
    return static_cast<int64_t>(values / grid_.size());
}

void evaluate_qhat(CollisionGpu& op, std::span<const std::complex<double>> fhat,
                   std::span<std::complex<double>> qhat) {
    const int64_t nc = op.cells(fhat.size());
    if (qhat.size() != fhat.size()) throw ConfigError("evaluate_qhat: fhat and qhat sizes differ");
    gpu_check(boltz_qhat_batch(op.handle(), reinterpret_cast<const double*>(fhat.data()),
                               reinterpret_cast<double*>(qhat.data()), nc, BOLTZ_MEM_HOST, nullptr),
              "evaluate_qhat");
}

void conserve(CollisionGpu& op, std::span<const double> q_raw, std::span<double> q) {
    const int64_t nc = op.cells(q_raw.size());
    if (q.size() != q_raw.size()) throw ConfigError("conserve: q_raw and q sizes differ");
    gpu_check(boltz_conserve_batch(op.handle(), q_raw.data(), q.data(), nc, BOLTZ_MEM_HOST, nullptr), "conserve");
}

void collide(CollisionGpu& op, std::span<const double> f, std::span<double> q, double epsilon,
             std::span<double> max_imag) {
    const int64_t nc = op.cells(f.size());
    if (q.size() != f.size()) throw ConfigError("collide: f and q sizes differ");
    if (!(epsilon > 0.0)) throw ConfigError("collide: epsilon must be positive");
    if (!max_imag.empty() && (int64_t)max_imag.size() != nc)
        throw ConfigError("collide: max_imag must hold one value per cell");
    gpu_check(boltz_collide_batch(op.handle(), f.data(), q.data(), nc, 1.0 / epsilon,
                                  max_imag.empty() ? nullptr : max_imag.data(), BOLTZ_MEM_HOST, nullptr),
              "collide");
}

void collision_rk2(CollisionGpu& op, std::span<double> cells, double dt, double epsilon) {
    const int64_t nc = op.cells(cells.size());
    if (!(dt > 0.0) || !(epsilon > 0.0)) throw ConfigError("collision_rk2: dt and epsilon must be positive");
    gpu_check(boltz_rk2_batch(op.handle(), cells.data(), nc, dt, 1.0 / epsilon, BOLTZ_MEM_HOST, nullptr),
              "collision_rk2");
}

}  // namespace boltz
