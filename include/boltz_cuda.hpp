// boltz_cuda.hpp -- header-only C++ view of the C ABI (boltz_cuda.h) in the
// shape of the reference's collision API, for the reference's C++ drivers
// (grid, time stepping) to call.  See INTEGRATION.md for the mapping onto
// boltz::ConfigError / IoError / NumericError (errors.hpp:8-35).
//
//   reference                                   here
//   SpectralTransform(grid)   fourier.hpp:31    CollisionOperator(n, L, kernel, table)
//   forward / inverse         fourier.hpp:36-41 forward / inverse (batched)
//   evaluate_qhat / conserve / collide          evaluate_qhat / conserve / collide (batched)
//   collision_rk2             SPEC.md:383       collision_rk2 (in place, batched)
#pragma once

#include <complex>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "boltz_cuda.h"

// Errors.  Built inside the reference tree (its include directory on the
// path, so <boltz/errors.hpp> resolves), failures are the reference's own
// exceptions: boltz::ConfigError / IoError / NumericError (errors.hpp:9-35), and
// CUDA / NCCL failures a boltz::Error of category 5; boltz::cuda::Error is then
// boltz::Error itself, so a reference strang_step that catches
// boltz::NumericError catches ours.  Standalone, boltz::cuda::Error
// is a std::runtime_error with the same integer categories.
#if !defined(BOLTZ_CUDA_STANDALONE_ERRORS) && __has_include(<boltz/errors.hpp>)
#include <boltz/errors.hpp>
#define BOLTZ_CUDA_REFERENCE_ERRORS 1
#endif

namespace boltz::cuda {

#if BOLTZ_CUDA_REFERENCE_ERRORS
using Error = boltz::Error;

[[noreturn]] inline void throw_error(int category, const std::string& what) {
    switch (category) {
        case BOLTZ_ERR_CONFIG: throw boltz::ConfigError(what);
        case BOLTZ_ERR_IO: throw boltz::IoError(what);
        case BOLTZ_ERR_NUMERIC: throw boltz::NumericError(what);
        default: throw boltz::Error(static_cast<boltz::ErrorCategory>(category), "CUDA: " + what);
    }
}
#else
// Category 2/3/4 as in boltz::ErrorCategory (errors.hpp:8-13); 5 = CUDA/NCCL.
class Error : public std::runtime_error {
public:
    Error(int category, const std::string& what) : std::runtime_error(what), category_(category) {}
    int category() const { return category_; }

private:
    int category_;
};

[[noreturn]] inline void throw_error(int category, const std::string& what) { throw Error(category, what); }
#endif

// the integer category of either error type (2/3/4 reference, 5 CUDA/NCCL)
inline int category_of(const Error& e) { return static_cast<int>(e.category()); }

inline void check(int rc) {
    if (rc != BOLTZ_OK) throw_error(rc, boltz_last_error());
}

struct Kernel {
    double lambda = 1.0;  // |u|^lambda
    double beta = 1.0;
    double r0 = 0.0;      // 0 -> r0 = L
};

// Host weight table, dense zeta-major N^6 doubles.
inline std::vector<double> generate_table(int n, double L, const Kernel& k, int panels = 64, int threads = 0) {
    std::vector<double> G(static_cast<size_t>(n) * n * n * n * n * n);
    check(boltz_generate_table(n, L, k.lambda, k.beta, k.r0 > 0 ? k.r0 : L, panels, G.data(), threads));
    return G;
}

class CollisionOperator {
public:
    CollisionOperator(int n, double L, const Kernel& k, std::span<const double> table, int device = 0) : n_(n) {
        if (table.size() != static_cast<size_t>(n) * n * n * n * n * n)
            throw_error(BOLTZ_ERR_CONFIG, "weight table size is not N^6");
        check(boltz_create(n, L, k.lambda, k.beta, k.r0 > 0 ? k.r0 : L, table.data(), device, &ctx_));
    }
    // the weights generated on the device (no N^6 host table)
    struct Generated {
        int panels = 64;
    };
    CollisionOperator(int n, double L, const Kernel& k, Generated g, int device = 0) : n_(n) {
        check(boltz_create_generated(n, L, k.lambda, k.beta, k.r0 > 0 ? k.r0 : L, g.panels, device, &ctx_));
    }
    ~CollisionOperator() { boltz_destroy(ctx_); }
    CollisionOperator(const CollisionOperator&) = delete;
    CollisionOperator& operator=(const CollisionOperator&) = delete;

    size_t cell_size() const { return static_cast<size_t>(n_) * n_ * n_; }

    // host spans: ncells = f.size() / N^3 consecutive cells (velocity_grid.hpp:30-32)
    void forward(std::span<const double> f, std::span<std::complex<double>> fhat) {
        check(boltz_forward_batch(ctx_, f.data(), reinterpret_cast<double*>(fhat.data()), cells(f.size()),
                                  BOLTZ_MEM_HOST, nullptr));
    }
    void inverse(std::span<const std::complex<double>> g, std::span<double> f, double* max_imag = nullptr) {
        check(boltz_inverse_batch(ctx_, reinterpret_cast<const double*>(g.data()), f.data(), max_imag,
                                  cells(g.size()), BOLTZ_MEM_HOST, nullptr));
    }
    void evaluate_qhat(std::span<const std::complex<double>> fhat, std::span<std::complex<double>> qhat) {
        check(boltz_qhat_batch(ctx_, reinterpret_cast<const double*>(fhat.data()), reinterpret_cast<double*>(qhat.data()),
                               cells(fhat.size()), BOLTZ_MEM_HOST, nullptr));
    }
    void conserve(std::span<const double> q_raw, std::span<double> q) {
        check(boltz_conserve_batch(ctx_, q_raw.data(), q.data(), cells(q_raw.size()), BOLTZ_MEM_HOST, nullptr));
    }
    void collide(std::span<const double> f, std::span<double> q, double epsilon, double* max_imag = nullptr) {
        if (!(epsilon > 0)) throw_error(BOLTZ_ERR_CONFIG, "collide: epsilon must be positive");
        check(boltz_collide_batch(ctx_, f.data(), q.data(), cells(f.size()), 1.0 / epsilon, max_imag, BOLTZ_MEM_HOST,
                                  nullptr));
    }
    void collision_rk2(std::span<double> field, double dt, double epsilon) {
        if (!(dt > 0 && epsilon > 0)) throw_error(BOLTZ_ERR_CONFIG, "collision_rk2: dt, epsilon must be positive");
        check(boltz_rk2_batch(ctx_, field.data(), cells(field.size()), dt, 1.0 / epsilon, BOLTZ_MEM_HOST, nullptr));
    }
    // device-pointer variants (ordered on `stream`)
    void collision_rk2_device(double* field, int64_t ncells, double dt, double epsilon, void* stream = nullptr) {
        check(boltz_rk2_batch(ctx_, field, ncells, dt, 1.0 / epsilon, BOLTZ_MEM_DEVICE, stream));
    }
    // compute_moments: 7 values per cell (rho, rho V, rho e, T, H)
    std::vector<double> moments(std::span<const double> f) {
        std::vector<double> out(7 * static_cast<size_t>(cells(f.size())));
        check(boltz_moments_batch(ctx_, f.data(), out.data(), cells(f.size()), BOLTZ_MEM_HOST, nullptr));
        return out;
    }
    // marginal_distribution g(v1): N values per cell
    std::vector<double> marginal(std::span<const double> f) {
        std::vector<double> out(static_cast<size_t>(n_) * cells(f.size()));
        check(boltz_marginal_batch(ctx_, f.data(), out.data(), cells(f.size()), BOLTZ_MEM_HOST, nullptr));
        return out;
    }
    boltz_ctx* handle() { return ctx_; }

private:
    int64_t cells(size_t values) const {
        if (values % cell_size()) throw_error(BOLTZ_ERR_CONFIG, "array is not a whole number of cells");
        return static_cast<int64_t>(values / cell_size());
    }
    int n_;
    boltz_ctx* ctx_ = nullptr;
};

}  // namespace boltz::cuda
