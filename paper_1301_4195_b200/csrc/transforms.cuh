// transforms.cuh -- K1 (batched forward 3D FFT) and K3 (inverse 3D FFT +
// conservation projection + RK2 epilogue) on the group layout.
//
// Reference semantics (fourier.hpp:11-22):
//   forward  fhat_k = (dv/sqrt(2pi))^3 * par * s_k * DFT_-[ s_m c_m f_m ]_k
//   inverse  f_k    = Re (dzeta/sqrt(2pi))^3 * par * s_k * DFT_+[ s_m g_m ]_k
// with s_m = (-1)^{m1+m2+m3}, par = ((-1)^{N/2})^3, c_m the trapezoid
// coefficients.  The inverse's input sign s_m is applied by the convolution
// epilogue (conv.cuh), so the inverse passes here start from s_m*Qhat_m.
#pragma once
#include "common.cuh"
#include "fft.cuh"

namespace boltz_gpu {

enum PassMode : int {
    PASS_PACK_FWD = 0,   // user real f -> s c f -> FFT(axis 2) -> group complex
    PASS_MID = 1,        // group complex FFT in place
    PASS_FWD_LAST = 2,   // FFT then * scale*par*s_k (axis 0)
    PASS_INV_LAST = 3,   // FFT then Re(scale*par*s_k*z) -> group real, max|Im|
};

// row -> (base index, stride) of a line along AXIS in a cell's N^3 block
template <int N, int AXIS>
__device__ __forceinline__ void line_of(int row, int& base, int& stride) {
    if (AXIS == 2) { base = row * N; stride = 1; }
    else if (AXIS == 1) { base = (row / N) * N * N + (row % N); stride = N; }
    else { base = row; stride = N * N; }
}

// blockDim = (32, R): threadIdx.x = lane (cell in group), threadIdx.y = line.
// grid = (ceil(N^2 / R), ngroups).
template <int N, int AXIS, int SIGN, int MODE>
__global__ void __launch_bounds__(256)
k_fft_pass(const double* __restrict__ fuser, double2* __restrict__ A, double* __restrict__ Rout,
           unsigned long long* __restrict__ maximag, int* __restrict__ flag, long long ncells,
           double scale) {
    constexpr int N3 = N * N * N;
    const int lane = threadIdx.x;
    const int row = blockIdx.x * blockDim.y + threadIdx.y;
    const long long g = blockIdx.y;
    const long long cell = g * kLanes + lane;
    double im_max = 0.0;
    if (row < N * N) {
        int base, stride;
        line_of<N, AXIS>(row, base, stride);
        double2 x[N];
        double2* Ag = A + (size_t)g * N3 * kLanes + lane;
        if (MODE == PASS_PACK_FWD) {
            const int i1 = row / N, i2 = row % N;
            const double cc = axis_coeff(N, i1) * axis_coeff(N, i2);
            const bool live = cell < ncells;
            const double* fc = fuser + (size_t)cell * N3 + base;
            bool bad = false;
#pragma unroll
            for (int j = 0; j < N; ++j) {
                double v = live ? fc[j] : 0.0;
                bad |= !isfinite(v);
                double s = ((i1 + i2 + j) & 1) ? -cc : cc;
                x[j] = make_double2(v * s * axis_coeff(N, j), 0.0);
            }
            if (bad) atomicOr(flag, 1);
        } else {
#pragma unroll
            for (int j = 0; j < N; ++j) x[j] = Ag[(size_t)(base + j * stride) * kLanes];
        }
        RegFFT<N, SIGN, N>::run(x);
        if (MODE == PASS_FWD_LAST) {
            // AXIS 0: row = i2*N + i3, element j has k1 = j
            const int rs = (row / N + row % N) & 1;
#pragma unroll
            for (int j = 0; j < N; ++j) {
                double s = ((rs + j) & 1) ? -scale : scale;
                Ag[(size_t)(base + j * stride) * kLanes] = make_double2(x[j].x * s, x[j].y * s);
            }
        } else if (MODE == PASS_INV_LAST) {
            const int rs = (row / N + row % N) & 1;
            double* Rg = Rout + (size_t)g * N3 * kLanes + lane;
#pragma unroll
            for (int j = 0; j < N; ++j) {
                double s = ((rs + j) & 1) ? -scale : scale;
                Rg[(size_t)(base + j * stride) * kLanes] = x[j].x * s;
                im_max = fmax(im_max, fabs(x[j].y * scale));
            }
        } else {
#pragma unroll
            for (int j = 0; j < N; ++j) Ag[(size_t)(base + j * stride) * kLanes] = x[j];
        }
    }
    if (MODE == PASS_INV_LAST) {
        // reduce over the block's lines, one atomic per cell (max is order-free)
        __shared__ double red[8][kLanes];
        red[threadIdx.y][lane] = im_max;
        __syncthreads();
        if (threadIdx.y == 0) {
            double m = red[0][lane];
            for (int r = 1; r < (int)blockDim.y; ++r) m = fmax(m, red[r][lane]);
            if (cell < ncells)
                atomicMax(maximag + cell, (unsigned long long)__double_as_longlong(m));
        }
    }
}

// K3 epilogue: conservation projection + RK2 axpy.
//   Q   = Qt - C^T (C C^T)^{-1} C Qt        (C rows: w, v1 w, v2 w, v3 w, |v|^2 w)
//   out = base + coef * Q    (base == nullptr -> out = coef * Q)
// Qt comes in the group layout (real), out/base are in the user layout [cell][N^3].
// ---- K3 epilogue for grids whose cube does not fit in shared memory (N = 32; also conserve()):
// two launches over (cell octet) x (node slice) blocks so that every SM works
// (one block per 32-cell group left most of the GPU idle: 10% of an N=24 step).
//   k_project_moments: partial moments of each slice   -> part[cell][slice][5]
//   k_project_apply:   fixed-order sum of the slices, lambda = (CC^T)^{-1} m,
//                      out = base + coef * (Qt - C^T lambda) on its slice
// Deterministic: fixed thread -> node assignment, fixed reduction order.
constexpr int kProjSlices = 8;

template <int N>
__device__ __forceinline__ void proj_row(int idx, const ProjConst& pc, double& w, double& v1, double& v2, double& v3) {
    const int i1 = idx / (N * N), i2 = (idx / N) % N, i3 = idx % N;
    v1 = pc.dv * (i1 - N / 2);
    v2 = pc.dv * (i2 - N / 2);
    v3 = pc.dv * (i3 - N / 2);
    w = axis_coeff(N, i1) * axis_coeff(N, i2) * axis_coeff(N, i3) * pc.dv * pc.dv * pc.dv;
}

// grid = (ngroups * 4, kProjSlices); block = 256 = 8 cells x 32 node strides
template <int N>
__global__ void __launch_bounds__(256)
k_project_moments(const double* __restrict__ R, double* __restrict__ part, long long ncells, ProjConst pc) {
    constexpr int N3 = N * N * N;
    constexpr int SL = (N3 + kProjSlices - 1) / kProjSlices;
    const long long g = blockIdx.x / 4;
    const int c = threadIdx.x & 7, j = threadIdx.x >> 3;
    const int lane = (blockIdx.x % 4) * 8 + c;
    const int idx0 = blockIdx.y * SL, idx1 = min(N3, idx0 + SL);
    double m[5] = {0, 0, 0, 0, 0};
    for (int idx = idx0 + j; idx < idx1; idx += 32) {
        double w, v1, v2, v3;
        proj_row<N>(idx, pc, w, v1, v2, v3);
        const double q = R[((size_t)g * N3 + idx) * kLanes + lane] * w;
        m[0] += q;
        m[1] += v1 * q;
        m[2] += v2 * q;
        m[3] += v3 * q;
        m[4] += (v1 * v1 + v2 * v2 + v3 * v3) * q;
    }
    __shared__ double red[5][32][8];
#pragma unroll
    for (int a = 0; a < 5; ++a) red[a][j][c] = m[a];
    __syncthreads();
    if (j < 5) {  // thread (c, a=j) sums the 32 strides of moment a in order
        double s = 0.0;
        for (int r = 0; r < 32; ++r) s += red[j][r][c];
        const long long cell = g * kLanes + lane;
        if (cell < ncells) part[((size_t)cell * kProjSlices + blockIdx.y) * 5 + j] = s;
    }
}

template <int N>
__global__ void __launch_bounds__(256)
k_project_apply(const double* __restrict__ R, const double* __restrict__ part, const double* __restrict__ base,
                double* __restrict__ out, long long ncells, double coef, ProjConst pc, int* __restrict__ flag) {
    constexpr int N3 = N * N * N;
    constexpr int SL = (N3 + kProjSlices - 1) / kProjSlices;
    const long long g = blockIdx.x / 4;
    const int c = threadIdx.x & 7, j = threadIdx.x >> 3;
    const int lane = (blockIdx.x % 4) * 8 + c;
    const long long cell = g * kLanes + lane;
    __shared__ double lam[8][5];
    if (j == 0) {
        double s[5] = {0, 0, 0, 0, 0};
        if (cell < ncells)
            for (int sl = 0; sl < kProjSlices; ++sl)
                for (int a = 0; a < 5; ++a) s[a] += part[((size_t)cell * kProjSlices + sl) * 5 + a];
        for (int a = 0; a < 5; ++a) {
            double t = 0.0;
            for (int b = 0; b < 5; ++b) t = fma(pc.ginv[a * 5 + b], s[b], t);
            lam[c][a] = t;
        }
    }
    __syncthreads();
    if (cell >= ncells) return;
    const int idx0 = blockIdx.y * SL, idx1 = min(N3, idx0 + SL);
    bool bad = false;
    for (int idx = idx0 + j; idx < idx1; idx += 32) {
        double w, v1, v2, v3;
        proj_row<N>(idx, pc, w, v1, v2, v3);
        const double cl = lam[c][0] + v1 * lam[c][1] + v2 * lam[c][2] + v3 * lam[c][3] +
                          (v1 * v1 + v2 * v2 + v3 * v3) * lam[c][4];
        const size_t o = (size_t)cell * N3 + idx;
        double v = coef * (R[((size_t)g * N3 + idx) * kLanes + lane] - w * cl);
        if (base) v += base[o];
        bad |= !isfinite(v);
        out[o] = v;
    }
    if (bad) atomicOr(flag, 2);
}

// ---- layout conversion kernels (API entry points only, not the RK2 path) ----

// user complex [cell][N^3] (interleaved) -> group complex, optional * s_m
template <int N>
__global__ void k_pack_complex(const double2* __restrict__ in, double2* __restrict__ A, long long ncells,
                               int apply_sign) {
    constexpr int N3 = N * N * N;
    const long long g = blockIdx.y;
    const int lane = threadIdx.x & 31;
    for (int idx = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); idx < N3;
         idx += gridDim.x * (blockDim.x >> 5)) {
        const long long cell = g * kLanes + lane;
        double2 v = cell < ncells ? in[(size_t)cell * N3 + idx] : make_double2(0.0, 0.0);
        if (apply_sign) {
            const int s = (idx / (N * N) + (idx / N) % N + idx % N) & 1;
            if (s) v = make_double2(-v.x, -v.y);
        }
        A[((size_t)g * N3 + idx) * kLanes + lane] = v;
    }
}

// group complex -> user complex, optional * s_k (undo the conv epilogue sign)
template <int N>
__global__ void k_unpack_complex(const double2* __restrict__ A, double2* __restrict__ out, long long ncells,
                                 int apply_sign) {
    constexpr int N3 = N * N * N;
    const long long g = blockIdx.y;
    const int lane = threadIdx.x & 31;
    for (int idx = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); idx < N3;
         idx += gridDim.x * (blockDim.x >> 5)) {
        const long long cell = g * kLanes + lane;
        if (cell >= ncells) continue;
        double2 v = A[((size_t)g * N3 + idx) * kLanes + lane];
        if (apply_sign) {
            const int s = (idx / (N * N) + (idx / N) % N + idx % N) & 1;
            if (s) v = make_double2(-v.x, -v.y);
        }
        out[(size_t)cell * N3 + idx] = v;
    }
}

// group real -> user real
template <int N>
__global__ void k_unpack_real(const double* __restrict__ R, double* __restrict__ out, long long ncells) {
    constexpr int N3 = N * N * N;
    const long long g = blockIdx.y;
    const int lane = threadIdx.x & 31;
    for (int idx = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); idx < N3;
         idx += gridDim.x * (blockDim.x >> 5)) {
        const long long cell = g * kLanes + lane;
        if (cell >= ncells) continue;
        out[(size_t)cell * N3 + idx] = R[((size_t)g * N3 + idx) * kLanes + lane];
    }
}

}  // namespace boltz_gpu

namespace boltz_gpu {
// user real -> group real
template <int N>
__global__ void k_pack_real(const double* __restrict__ in, double* __restrict__ R, long long ncells) {
    constexpr int N3 = N * N * N;
    const long long g = blockIdx.y;
    const int lane = threadIdx.x & 31;
    for (int idx = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); idx < N3;
         idx += gridDim.x * (blockDim.x >> 5)) {
        const long long cell = g * kLanes + lane;
        R[((size_t)g * N3 + idx) * kLanes + lane] = cell < ncells ? in[(size_t)cell * N3 + idx] : 0.0;
    }
}
}  // namespace boltz_gpu
