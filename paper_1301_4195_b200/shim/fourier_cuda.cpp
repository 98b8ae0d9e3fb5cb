// boltz::SpectralTransform on the B200, against the reference's UNMODIFIED
// header proj/include/boltz/fourier.hpp:28-52 -- the drop-in a maintainer
// compiles into the reference tree in place of the (absent, FFTW-backed)
// src/fourier.cpp (CMakeLists.txt:22).
//
//   fourier.hpp                      here
//   SpectralTransform(grid)   :31    boltz_create_transform(N, L) -- a device
//                                    context with no weight table; it lives in
//                                    plan_fwd_ (the header's FFTW plan slot)
//   ~SpectralTransform()      :32    boltz_destroy
//   forward(f, fhat)          :36    boltz_forward_batch (one cell, host spans)
//   inverse(g, f, max_imag)   :38-41 boltz_inverse_batch (Re part, max |Im|)
//
// Conventions are the header's (fourier.hpp:11-22): trapezoid-weighted
// forward, plain-lattice-sum inverse, phase wrapping by (-1)^m, (-1)^k and
// ((-1)^{N/2})^3 -- computed by the library's K1/K3 kernels.  Errors are the
// reference's exceptions (errors.hpp:9-35).  Like the FFTW version, an
// instance is not thread-safe; distinct instances (distinct device contexts)
// may run concurrently (fourier.hpp:24-25).  BOLTZ_DEVICE selects the GPU
// (default 0).
#include <complex>
#include <cstdlib>
#include <span>
#include <string>

#include "boltz/errors.hpp"
#include "boltz/fourier.hpp"
#include "boltz_cuda.h"

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

int device_ordinal() {
    const char* e = std::getenv("BOLTZ_DEVICE");
    return e ? std::atoi(e) : 0;
}

boltz_ctx* ctx_of(void* p) { return static_cast<boltz_ctx*>(p); }

}  // namespace

SpectralTransform::SpectralTransform(const VelocityGrid& grid) : grid_(grid) {
    const int n = grid.n;
    // the header's phase tables (fourier.hpp:49-50), kept so the object holds
    // what its declaration says; the device kernels apply the same factors
    sign_.resize(grid.size());
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            for (int k = 0; k < n; ++k) sign_[grid.flat(i, j, k)] = ((i + j + k) & 1) ? -1.0 : 1.0;
    parity_const_ = ((n / 2) & 1) ? -1.0 : 1.0;
    boltz_ctx* c = nullptr;
    gpu_check(boltz_create_transform(n, grid.half_width, device_ordinal(), &c), "SpectralTransform");
    plan_fwd_ = c;  // one device context serves both directions
    plan_bwd_ = c;
}

SpectralTransform::~SpectralTransform() {
    boltz_destroy(ctx_of(plan_fwd_));
    plan_fwd_ = plan_bwd_ = nullptr;
}

void SpectralTransform::forward(std::span<const double> f, std::span<std::complex<double>> fhat) {
    if (f.size() != grid_.size() || fhat.size() != grid_.size())
        throw ConfigError("SpectralTransform::forward: spans must hold N^3 values");
    gpu_check(boltz_forward_batch(ctx_of(plan_fwd_), f.data(), reinterpret_cast<double*>(fhat.data()), 1,
                                  BOLTZ_MEM_HOST, nullptr),
              "SpectralTransform::forward");
}

void SpectralTransform::inverse(std::span<const std::complex<double>> g, std::span<double> f, double* max_imag) {
    if (g.size() != grid_.size() || f.size() != grid_.size())
        throw ConfigError("SpectralTransform::inverse: spans must hold N^3 values");
    double mi = 0.0;
    gpu_check(boltz_inverse_batch(ctx_of(plan_bwd_), reinterpret_cast<const double*>(g.data()), f.data(), &mi, 1,
                                  BOLTZ_MEM_HOST, nullptr),
              "SpectralTransform::inverse");
    if (max_imag) *max_imag = mi;
}

}  // namespace boltz
