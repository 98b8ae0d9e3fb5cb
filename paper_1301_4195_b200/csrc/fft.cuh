// fft.cuh -- fully unrolled in-register 1D FFT of a length-N complex row.
//
// Replaces the FFTW plans of the reference's SpectralTransform
// (fourier.hpp:24-27,50-51).  One thread transforms one row of one cell; the
// batched 3D transform is three such passes over the group layout (one per
// axis), so every load/store is a coalesced 512 B warp transaction and the
// butterflies never touch shared memory.  Mixed radix 2/3 covers every
// supported N (4, 6, 8, 12, 16, 24, 32).  Twiddles come from the constant
// bank with compile-time indices (warp-uniform, no divergence).
#pragma once
#include "common.cuh"

namespace boltz_gpu {

__constant__ double2 c_tw[kTwTotal];  // single translation unit (boltz_cuda.cu)

// w_N^j for the top-level table of size TN, SIGN=-1 forward, +1 inverse.
template <int TN, int SIGN>
__device__ __forceinline__ double2 tw(int j) {
    double2 w = c_tw[tw_offset(TN) + (j % TN)];
    if (SIGN > 0) w.y = -w.y;
    return w;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// In-place DFT X[k] = sum_j x[j] w^{jk}, w = exp(SIGN*2*pi*i/N); TN = size of
// the top-level transform (selects the twiddle table).
template <int N, int SIGN, int TN>
struct RegFFT {
    __device__ __forceinline__ static void run(double2 (&x)[N]) {
        if constexpr (N == 1) {
            return;
        } else if constexpr (N == 2) {
            double2 a = x[0], b = x[1];
            x[0] = make_double2(a.x + b.x, a.y + b.y);
            x[1] = make_double2(a.x - b.x, a.y - b.y);
        } else if constexpr (N == 3) {
            // w = exp(SIGN 2 pi i/3) = (-1/2, SIGN*sqrt(3)/2)
            const double2 w1 = tw<TN, SIGN>(TN / 3);
            double2 a = x[0], b = x[1], c = x[2];
            double sx = b.x + c.x, sy = b.y + c.y;   // b + c
            double dx = b.x - c.x, dy = b.y - c.y;   // b - c
            x[0] = make_double2(a.x + sx, a.y + sy);
            // X1 = a + w b + w^2 c = a - (b+c)/2 + i*Im(w)*(b-c)
            double rx = fma(-0.5, sx, a.x), ry = fma(-0.5, sy, a.y);
            x[1] = make_double2(fma(-w1.y, dy, rx), fma(w1.y, dx, ry));
            x[2] = make_double2(fma(w1.y, dy, rx), fma(-w1.y, dx, ry));
        } else {
            static_assert(N % 2 == 0, "supported sizes are 2^a * 3");
            double2 e[N / 2], o[N / 2];
#pragma unroll
            for (int j = 0; j < N / 2; ++j) { e[j] = x[2 * j]; o[j] = x[2 * j + 1]; }
            RegFFT<N / 2, SIGN, TN>::run(e);
            RegFFT<N / 2, SIGN, TN>::run(o);
#pragma unroll
            for (int k = 0; k < N / 2; ++k) {
                double2 t;
                if (k == 0) t = o[k];
                else if (4 * k == N) t = SIGN < 0 ? make_double2(o[k].y, -o[k].x)   // * (-i)
                                                   : make_double2(-o[k].y, o[k].x); // * (+i)
                else t = cmul(o[k], tw<TN, SIGN>(k * (TN / N)));
                x[k] = make_double2(e[k].x + t.x, e[k].y + t.y);
                x[k + N / 2] = make_double2(e[k].x - t.x, e[k].y - t.y);
            }
        }
    }
};

}  // namespace boltz_gpu
