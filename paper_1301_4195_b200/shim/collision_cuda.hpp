// The reference's collision operations on the B200,
// in the reference's own types: boltz::VelocityGrid (velocity_grid.hpp:17-47),
// std::span / std::complex<double> data (fourier.hpp:36-41) and the
// boltz::ConfigError / IoError / NumericError exceptions (errors.hpp:9-35).
// Compiled into the reference tree beside shim/fourier_cuda.cpp; the
// reference's own collision.cpp / weights.cpp are absent
// (CMakeLists.txt:22-33), so the SPEC's operation names are kept and the
// per-cell workspace (SPEC CollisionWorkspace) becomes the device context.
//
//   SPEC operation                                  here
//   evaluate_qhat(grid, table, fhat)   SPEC:186    evaluate_qhat(op, fhat, qhat)
//   conserve(op, q_raw)                SPEC:204    conserve(op, q_raw, q)
//   collide(grid, table, ws, f, eps)   SPEC:195    collide(op, f, q, eps, max_imag)
//   collision_rk2(field, dt)           SPEC:383    collision_rk2(op, cells, dt, eps)
//
// Every span holds a whole number of N^3 cells (flat index (i*N+j)*N+k,
// velocity_grid.hpp:30-32); a call over many cells is ONE batched GPU call.
#pragma once

#include <complex>
#include <cstdint>
#include <span>
#include <vector>

#include "boltz/velocity_grid.hpp"
#include "boltz_cuda.h"

namespace boltz {

// KernelSpec of the weights module: |u|^lambda, beta, r0
// (r0 <= 0 means r0 = L).
struct GpuKernelSpec {
    double lambda = 1.0;
    double beta = 1.0;
    double r0 = 0.0;
};

// The weight table resident in HBM (folded from the caller's dense zeta-major
// G) plus the device workspace.  Not copyable; not thread-safe
// (one per worker thread / GPU, like the reference's workspaces).
class CollisionGpu {
public:
    // G: the dense N^6 table of generate_table / load_table
    CollisionGpu(const VelocityGrid& grid, const GpuKernelSpec& k, std::span<const double> G, int device = 0);
    // the same weights evaluated on the device (no host table)
    CollisionGpu(const VelocityGrid& grid, const GpuKernelSpec& k, int device = 0);
    ~CollisionGpu();
    CollisionGpu(const CollisionGpu&) = delete;
    CollisionGpu& operator=(const CollisionGpu&) = delete;

    const VelocityGrid& grid() const { return grid_; }
    boltz_ctx* handle() { return ctx_; }
    int64_t cells(std::size_t values) const;  // ConfigError unless a whole number of cells

private:
    const VelocityGrid& grid_;
    boltz_ctx* ctx_ = nullptr;
};

void evaluate_qhat(CollisionGpu& op, std::span<const std::complex<double>> fhat,
                   std::span<std::complex<double>> qhat);
void conserve(CollisionGpu& op, std::span<const double> q_raw, std::span<double> q);
// q = (1/epsilon) P_N(Q~(f)); NumericError on non-finite input
void collide(CollisionGpu& op, std::span<const double> f, std::span<double> q, double epsilon,
             std::span<double> max_imag = {});
// midpoint RK2 in place on every cell; NumericError on a
// non-finite input or stage
void collision_rk2(CollisionGpu& op, std::span<double> cells, double dt, double epsilon = 1.0);

}  // namespace boltz
