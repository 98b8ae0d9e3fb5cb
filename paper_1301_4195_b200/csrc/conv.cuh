// conv.cuh -- K2: the O(N^6) weighted Fourier-space convolution
//   Qhat(zeta_k) = sum_m G(xi_m, zeta_k) fhat(xi_m) fhat(zeta_k - xi_m) omega_m
// ("the hot loop of the whole program",
// SPEC.md:155), on FP64 CUDA cores.
//
// Structure:
//  * Per axis the shifted index is s = k - m + N/2 (kept only in [0,N)), so for
//    an output row (k1,k2) and an input row (m1,m2) the inner sum over
//    (k3, m3) is a 1D band: out[k3] += H[k3][m3] * x[m3] * y[k3-m3+N/2] with
//    x = fhat(m1,m2,:), y = fhat(s1,s2,:).
//  * Pair symmetry: m -> sigma(m) = k - m + N/2 (all three axes) is an
//    involution of the valid set that swaps the two fhat factors, so
//    Qhat(k) = sum over orbit representatives of [G'(k,m)+G'(k,sigma m)]
//    fhat(m) fhat(sigma m), G' = G*omega.  Only representative input rows are
//    visited (half of them); the self-paired row keeps its m3 <= s3 half.  The
//    folded table H is built once per context from the caller's G.
//  * lane == cell (group layout), so H is warp-uniform: one 16 B load feeds
//    two terms for 32 cells.  Each thread keeps a T-wide k3 chunk of
//    accumulators and a T-wide window of y in registers; x is loaded once per
//    diagonal.  Every (k3, m3) index is a compile-time constant after unroll.
//  * Deterministic: each output is accumulated by one thread in a fixed order
//    (SPEC.md:233); results are independent of batch composition.
#pragma once
#include "common.cuh"

namespace boltz_gpu {

// ---- band enumeration shared by the kernel (compile time) and the host table
// builder (run time).  Tile (kc, sc): k3 in [kc*T, kc*T+T), s3 in [sc*T, sc*T+T),
// m3 = k3 - s3 + N/2 must lie in [0, N).  Order: sc, then m3 ascending, then k3.
__host__ __device__ constexpr bool band_term(int n, int t, int kc, int sc, int m3, int kk) {
    int k3 = kc * t + kk, s3 = k3 - m3 + n / 2;
    return s3 >= sc * t && s3 < sc * t + t;
}
__host__ __device__ constexpr int band_kc_terms(int n, int t, int kc) {
    int c = 0;
    for (int sc = 0; sc < n / t; ++sc)
        for (int m3 = 0; m3 < n; ++m3)
            for (int kk = 0; kk < t; ++kk) c += band_term(n, t, kc, sc, m3, kk) ? 1 : 0;
    return c;
}
__host__ __device__ constexpr int band_slab_kc(int n, int t) {
    int mx = 0;
    for (int kc = 0; kc < n / t; ++kc) mx = band_kc_terms(n, t, kc) > mx ? band_kc_terms(n, t, kc) : mx;
    return (mx + 1) & ~1;  // even -> 16 B aligned double2 reads
}

// register tile width per N (accumulators + y window = 8T registers)
__host__ __device__ constexpr int conv_tile(int n) { return n == 24 ? 12 : (n == 32 ? 16 : n); }
#ifndef BOLTZ_CONV_WARPS
#define BOLTZ_CONV_WARPS 4
#endif
#ifndef BOLTZ_CONV_MINB
#define BOLTZ_CONV_MINB 1
#endif
#ifndef BOLTZ_CONV_PREFETCH
#define BOLTZ_CONV_PREFETCH 0
#endif
#ifndef BOLTZ_CONV_PIPE
#define BOLTZ_CONV_PIPE 1  // cp.async-pipelined kernel for N <= 16
#endif
constexpr int kConvWarps = BOLTZ_CONV_WARPS;  // cell groups per CTA (share the H stream via L1)

template <int N, int T, int KC>
__device__ __forceinline__ void conv_rows(const double2* __restrict__ Ag, const double* __restrict__ H,
                                          const int2* __restrict__ ent, int e0, int e1, double2 (&acc)[T]) {
    constexpr int NK = N / T;
    constexpr int SLAB_KC = band_slab_kc(N, T);
    constexpr int SLAB = NK * SLAB_KC;
    for (int e = e0; e < e1; ++e) {
        const int2 en = __ldg(ent + e);
#if BOLTZ_CONV_PREFETCH
        if (e + 1 < e1) {  // pull the next row pair into L1 while this one computes
            const int2 nx = __ldg(ent + e + 1);
            const double2* Xn = Ag + (size_t)nx.x * kLanes;
            const double2* Yn = Ag + (size_t)nx.y * kLanes;
#pragma unroll
            for (int j = 0; j < N; ++j) {
                asm volatile("prefetch.global.L1 [%0];" ::"l"(Xn + (size_t)j * kLanes));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(Yn + (size_t)j * kLanes));
            }
        }
#endif
        const double2* X = Ag + (size_t)en.x * kLanes;
        const double2* Y = Ag + (size_t)en.y * kLanes;
        const double2* Hs = reinterpret_cast<const double2*>(H + (size_t)e * SLAB + KC * SLAB_KC);
        int p = 0;
        double2 hb = make_double2(0.0, 0.0);
#pragma unroll
        for (int sc = 0; sc < NK; ++sc) {
            double2 y[T];
#pragma unroll
            for (int j = 0; j < T; ++j) y[j] = ldg2(Y + (size_t)(sc * T + j) * kLanes);
#pragma unroll
            for (int m3 = 0; m3 < N; ++m3) {
                bool any = false;
#pragma unroll
                for (int kk = 0; kk < T; ++kk) any |= band_term(N, T, KC, sc, m3, kk);
                if (!any) continue;
                const double2 xm = ldg2(X + (size_t)m3 * kLanes);
#pragma unroll
                for (int kk = 0; kk < T; ++kk) {
                    if (!band_term(N, T, KC, sc, m3, kk)) continue;
                    const int j = KC * T + kk - m3 + N / 2 - sc * T;  // y window slot
                    double h;
                    if ((p & 1) == 0) { hb = ldg2(Hs + (p >> 1)); h = hb.x; }
                    else h = hb.y;
                    ++p;
                    const double tr = fma(xm.x, y[j].x, -xm.y * y[j].y);
                    const double ti = fma(xm.x, y[j].y, xm.y * y[j].x);
                    acc[kk].x = fma(h, tr, acc[kk].x);
                    acc[kk].y = fma(h, ti, acc[kk].y);
                }
            }
        }
    }
}

// grid = (N*N*NK, ceil(ngroups / W)); block = 32*W.  Output B carries the
// inverse transform's input sign s_k (transforms.cuh).
template <int N>
__global__ void __launch_bounds__(kLanes* kConvWarps, BOLTZ_CONV_MINB)
k_conv(const double2* __restrict__ A, double2* __restrict__ B, const double* __restrict__ H,
       const int2* __restrict__ ent, const int* __restrict__ row_start, int ngroups) {
    constexpr int T = conv_tile(N);
    constexpr int NK = N / T;
    constexpr int N3 = N * N * N;
    const int kc = blockIdx.x % NK;
    const int row = blockIdx.x / NK;
    const int lane = threadIdx.x & 31;
    const int g = blockIdx.y * kConvWarps + (threadIdx.x >> 5);
    if (g >= ngroups) return;
    const double2* Ag = A + (size_t)g * N3 * kLanes + lane;
    double2 acc[T];
#pragma unroll
    for (int i = 0; i < T; ++i) acc[i] = make_double2(0.0, 0.0);
    const int e0 = __ldg(row_start + row), e1 = __ldg(row_start + row + 1);
    if (kc == 0) conv_rows<N, T, 0>(Ag, H, ent, e0, e1, acc);
    else if constexpr (NK > 1) conv_rows<N, T, (NK > 1 ? 1 : 0)>(Ag, H, ent, e0, e1, acc);
    const int k1 = row / N, k2 = row % N;
    double2* Bg = B + ((size_t)g * N3 + (size_t)row * N) * kLanes + lane;
#pragma unroll
    for (int kk = 0; kk < T; ++kk) {
        const int k3 = kc * T + kk;
        const double s = ((k1 + k2 + k3) & 1) ? -1.0 : 1.0;
        Bg[(size_t)k3 * kLanes] = make_double2(s * acc[kk].x, s * acc[kk].y);
    }
}

// ---------------------------------------------------------------------------
// K2, pipelined variant for a single register tile (T == N, i.e. N <= 16).
// Each warp owns a private shared-memory ring: while row pair e is computed
// from registers (y, accumulators) and shared memory (x, H), cp.async streams
// row pair e+1's x row, y row and H slab in behind it, so no global-memory
// latency is exposed at row boundaries (the stall that bounded k_conv).
//   per warp: x[2][N][32] + y[N][32] double2, H[2][SLAB] double
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int N>
struct PipeLayout {
    static constexpr int SLAB = band_slab_kc(N, N);                   // doubles, even
    static constexpr int X_BYTES = N * kLanes * 16;                   // one row of 32 cells
    static constexpr int H_BYTES = SLAB * 8;
    static constexpr int WARP_BYTES = 3 * X_BYTES + 2 * H_BYTES;      // x[2], y, H[2]
};

template <int N>
__device__ __forceinline__ void pipe_issue(char* wsm, int buf, const double2* __restrict__ Ag, const double* H,
                                           int2 en, int e, int lane) {
    using PL = PipeLayout<N>;
    double2* xs = reinterpret_cast<double2*>(wsm + buf * PL::X_BYTES);
    double2* ys = reinterpret_cast<double2*>(wsm + 2 * PL::X_BYTES);
    char* hs = wsm + 3 * PL::X_BYTES + buf * PL::H_BYTES;
    const double2* X = Ag + (size_t)en.x * kLanes;
    const double2* Y = Ag + (size_t)en.y * kLanes;
#pragma unroll
    for (int j = 0; j < N; ++j) {
        cp_async16(xs + j * kLanes + lane, X + (size_t)j * kLanes);
        cp_async16(ys + j * kLanes + lane, Y + (size_t)j * kLanes);
    }
    const char* hg = reinterpret_cast<const char*>(H + (size_t)e * PL::SLAB);
    for (int o = lane * 16; o < PL::H_BYTES; o += kLanes * 16) cp_async16(hs + o, hg + o);
    cp_async_commit();
}

template <int N>
__global__ void __launch_bounds__(kLanes* kConvWarps, 1)
k_conv_pipe(const double2* __restrict__ A, double2* __restrict__ B, const double* __restrict__ H,
            const int2* __restrict__ ent, const int* __restrict__ row_start, int ngroups) {
    using PL = PipeLayout<N>;
    constexpr int N3 = N * N * N;
    extern __shared__ __align__(16) char smem[];
    const int row = blockIdx.x;
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    const int g = blockIdx.y * kConvWarps + wid;
    if (g >= ngroups) return;  // whole warp exits together; warps never sync across each other
    char* wsm = smem + wid * PL::WARP_BYTES;
    const double2* Ag = A + (size_t)g * N3 * kLanes + lane;
    const double2* ys = reinterpret_cast<const double2*>(wsm + 2 * PL::X_BYTES);
    double2 acc[N];
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = make_double2(0.0, 0.0);
    const int e0 = __ldg(row_start + row), e1 = __ldg(row_start + row + 1);
    double2 y[N];
    if (e0 < e1) {
        pipe_issue<N>(wsm, 0, Ag, H, __ldg(ent + e0), e0, lane);
        cp_async_wait_all();
        __syncwarp();
#pragma unroll
        for (int j = 0; j < N; ++j) y[j] = ys[j * kLanes + lane];
    }
    for (int e = e0; e < e1; ++e) {
        const int cur = (e - e0) & 1;
        __syncwarp();  // every lane is done reading the buffers the next issue overwrites
        if (e + 1 < e1) pipe_issue<N>(wsm, cur ^ 1, Ag, H, __ldg(ent + e + 1), e + 1, lane);
        const double2* xs = reinterpret_cast<const double2*>(wsm + cur * PL::X_BYTES);
        const double2* hs = reinterpret_cast<const double2*>(wsm + 3 * PL::X_BYTES + cur * PL::H_BYTES);
        int p = 0;
        double2 hb = make_double2(0.0, 0.0);
#pragma unroll
        for (int m3 = 0; m3 < N; ++m3) {
            const double2 xm = xs[m3 * kLanes + lane];
#pragma unroll
            for (int kk = 0; kk < N; ++kk) {
                if (!band_term(N, N, 0, 0, m3, kk)) continue;
                const int j = kk - m3 + N / 2;
                double h;
                if ((p & 1) == 0) { hb = hs[p >> 1]; h = hb.x; }
                else h = hb.y;
                ++p;
                const double tr = fma(xm.x, y[j].x, -xm.y * y[j].y);
                const double ti = fma(xm.x, y[j].y, xm.y * y[j].x);
                acc[kk].x = fma(h, tr, acc[kk].x);
                acc[kk].y = fma(h, ti, acc[kk].y);
            }
        }
        if (e + 1 < e1) {
            cp_async_wait_all();
            __syncwarp();
#pragma unroll
            for (int j = 0; j < N; ++j) y[j] = ys[j * kLanes + lane];
        }
    }
    const int k1 = row / N, k2 = row % N;
    double2* Bg = B + ((size_t)g * N3 + (size_t)row * N) * kLanes + lane;
#pragma unroll
    for (int kk = 0; kk < N; ++kk) {
        const double s = ((k1 + k2 + kk) & 1) ? -1.0 : 1.0;
        Bg[(size_t)kk * kLanes] = make_double2(s * acc[kk].x, s * acc[kk].y);
    }
}

// ---- H table builder: H[e][slab pos] from one k1-plane of the caller's dense
// zeta-major G: Gk1[(k2*N + k3) * N^3 + m].  Entry e = output
// row (k1,k2) x representative input row (m1,m2).  term[pos] = (k3, m3) or
// (-1,-1) for padding.  omega_m = c3(m) dzeta^3 (velocity_grid.hpp:43-46).
__global__ void k_build_H(const double* __restrict__ Gk1, double* __restrict__ H, const int4* __restrict__ entk,
                          const short2* __restrict__ term, int e_begin, int e_end, int slab, int n, double w3) {
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long total = (long long)(e_end - e_begin) * slab;
    if (tid >= total) return;
    const int e = e_begin + (int)(tid / slab);
    const int pos = (int)(tid % slab);
    const int4 q = entk[e];  // k1, k2, m1, m2
    const short2 km = term[pos];
    double out = 0.0;
    if (km.x >= 0) {
        const int h = n / 2;
        const int k2 = q.y, m1 = q.z, m2 = q.w, k3 = km.x, m3 = km.y;
        const int s1 = q.x - m1 + h, s2 = k2 - m2 + h, s3 = k3 - m3 + h;
        const long long n3 = (long long)n * n * n;
        const double* Gk = Gk1 + ((long long)k2 * n + k3) * n3;
        const long long mf = ((long long)m1 * n + m2) * n + m3;
        const long long sf = ((long long)s1 * n + s2) * n + s3;
        const double wm = axis_coeff(n, m1) * axis_coeff(n, m2) * axis_coeff(n, m3) * w3;
        const double ws = axis_coeff(n, s1) * axis_coeff(n, s2) * axis_coeff(n, s3) * w3;
        const bool self_row = (m1 == s1) && (m2 == s2);
        if (!self_row || m3 < s3) out = Gk[mf] * wm + Gk[sf] * ws;
        else if (m3 == s3) out = Gk[mf] * wm;
    }
    H[(size_t)e * slab + pos] = out;
}

}  // namespace boltz_gpu
