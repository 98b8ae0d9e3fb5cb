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
//  * lane == cell (group layout), so H is warp-uniform: one 16 B broadcast
//    feeds two terms for 32 cells.  A thread keeps a T-wide chunk of k3
//    accumulators and a T-wide chunk of y in registers; x is read once per
//    diagonal.  Every (k3, m3) index is a compile-time constant after unroll.
//  * Deterministic: each output is accumulated by one thread in a fixed order
//    (SPEC.md:233); results are independent of batch composition.
//
// Kernels (per-N choice by measurement, see conv_kernel_for):
//  evaluate_qhat (any fhat) -- the plain pair-symmetric fold:
//  k_conv_pipe  N <= 16: per-warp TMA ring -- the next row pair's x row, y row
//               and H slab stream into shared memory while the current one
//               computes.
//  k_conv_kcs   N = 24, 32: one kernel per k-chunk (halves the unrolled code);
//               y row and H slab staged one row ahead (H is DRAM-resident at
//               N=32), x read from L2.
//  k_conv       no staging, direct loads: the plain statement of the order.
//  collide / RK2 (fhat of a real f) -- the Hermitian mirror schedule:
//  k_conv_mirror2  N = 8..16 (default): row-pair items, REST and the partner
//               row's REST' accumulated in TMEM; k_conv_mirror without TMEM.
//  k_conv_kcsm  N = 24, 32: phases per k-chunk (A of the pair leaders; FULL;
//               REST at N = 24), the chunk-0 kernels at N = 32 in the Gauss
//               5-instruction term form; k_conv_kcsr: N = 32's REST entries for
//               both k-chunks in one launch.
//  small batches: k_conv_seg (+ reduce; rows split over warps) and k_conv_cell
//               (lane = output k3, one or a few cells).
#pragma once
#include "common.cuh"

namespace boltz_gpu {

#include <type_traits>

// ---------------------------------------------------------------------------
// Band enumeration shared by the kernels (compile time) and the host table
// builder (run time).  Tile (kc, sc): k3 in [kc*T, kc*T+T), s3 in [sc*T, sc*T+T),
// m3 = k3 - s3 + N/2 in [0, N).  Within a k-chunk, tiles are visited in order
// t = 0..NK-1 and diagonals m3 in the order band_diag(); terms in k3 order.
// For NK == 2 the triangle tile comes first and the square tile (sc == kc,
// which covers every diagonal the row uses) last, walked so that the
// diagonals the next row's first tile needs are finished first (an x-slot
// refill schedule; measured in round 1, the order is kept for all kernels).
// ---------------------------------------------------------------------------
__host__ __device__ constexpr bool band_term(int n, int t, int kc, int sc, int m3, int kk) {
    int k3 = kc * t + kk, s3 = k3 - m3 + n / 2;
    return s3 >= sc * t && s3 < sc * t + t;
}
__host__ __device__ constexpr int band_tile_sc(int nk, int kc, int ti) { return nk == 2 ? (ti == 0 ? 1 - kc : kc) : ti; }
#ifndef BOLTZ_DIAG_REV
#define BOLTZ_DIAG_REV 1  // the chunk-1 square tile walks its diagonals in reverse (x-slot refill order)
#endif
__host__ __device__ constexpr int band_diag(int n, int nk, int kc, int ti, int i) {
    return (BOLTZ_DIAG_REV && nk == 2 && ti == 1 && kc == 1) ? n - 1 - i : i;
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
// does diagonal m3 carry any term of tile (kc, sc)?
__host__ __device__ constexpr bool diag_used(int n, int t, int kc, int sc, int m3) {
    bool any = false;
    for (int kk = 0; kk < t; ++kk) any = any || band_term(n, t, kc, sc, m3, kk);
    return any;
}

// ---------------------------------------------------------------------------
// Band types of the Hermitian mirror schedule (k_conv_mirror).  For real f,
// fhat(N-m) = conj fhat(m) (index mirror per axis) and G(N-k, N-m) = G(k, m)
// (G depends on |zeta|, |xi|, |xi - beta zeta/2|).  A folded term (k, {m, s})
// whose six indices m_a, s_a all lie in [2, N-2] -- where both trapezoid
// weights are 1 -- is the complex conjugate of its mirror term (N-k, {N-m,
// N-s}).  So the interior part of output row k is summed once and written,
// conjugated and k3-reversed, into row N-k as well.
//   BT_FULL every band term (in the mirror table: the A terms, then the REST terms)
//   BT_A    interior terms (m3, s3 in [2, N-2]) with k3 >= 1: these are mirrored
//   BT_REST the others: non-interior terms and the k3 = 0 column, whose mirror
//           (k3 = N) does not exist -- summed directly, for r and for N - r
// (the kernel unrolls the two typed bands only: a FULL entry runs both)
// ---------------------------------------------------------------------------
enum BandType { BT_FULL = 0, BT_A = 1, BT_REST = 2 };
constexpr int kBandTypes = 3;
__host__ __device__ constexpr bool mirror_interior(int n, int a) { return a >= 2 && a <= n - 2; }
__host__ __device__ constexpr bool type_term(int n, int ty, int k3, int m3) {
    const int s3 = k3 - m3 + n / 2;
    const bool mirrored = mirror_interior(n, m3) && mirror_interior(n, s3) && k3 != 0;
    return ty == BT_FULL ? true : ty == BT_A ? mirrored : !mirrored;
}
__host__ __device__ constexpr bool band_term_t(int n, int t, int kc, int sc, int m3, int kk, int ty) {
    return band_term(n, t, kc, sc, m3, kk) && type_term(n, ty, kc * t + kk, m3);
}
__host__ __device__ constexpr bool diag_used_t(int n, int t, int kc, int sc, int m3, int ty) {
    bool any = false;
    for (int kk = 0; kk < t; ++kk) any = any || band_term_t(n, t, kc, sc, m3, kk, ty);
    return any;
}
// H slab length (even) of one single-tile (T == N) entry of band type ty
__host__ __device__ constexpr int band_slab_type(int n, int ty) {
    int c = 0;
    for (int m3 = 0; m3 < n; ++m3)
        for (int kk = 0; kk < n; ++kk) c += band_term_t(n, n, 0, 0, m3, kk, ty) ? 1 : 0;
    return (c + 1) & ~1;
}
// H slab length of a mirror-table entry: a BT_FULL entry holds its A terms,
// then its REST terms, and runs as the two typed bands back to back (one copy
// of the unrolled term code instead of three)
__host__ __device__ constexpr int mirror_slab(int n, int ty) {
    return ty == BT_FULL ? band_slab_type(n, BT_A) + band_slab_type(n, BT_REST) : band_slab_type(n, ty);
}

// Register tile width and kernel per N, chosen by measurement on B200
// (scripts/dev/ab_conv.py, scripts/dev/ab_n32.sh; algorithmic TFLOP/s, round 1):
//   N=16: T=16 k_conv_pipe 47.5 | T=16 kcs 46.4 | T=8 kcs 39.7 | T=16 k_conv 41.1
//   N=24: T=24 kcs 45.5         | T=12 kcs 43.5 | T=24 pipe 36.0 | T=12 k_conv 34.3
//   N=32: T=16 kcs 45.3         | T=16 k_conv 33.3 | pipe 28.8
// (two removed variants also lost: a single-x-buffer streaming kernel with
//  T = N/2, 42.4 / 39.1 / 26.7, and k_conv split per k-chunk, 35.2 at N=32)
#ifndef BOLTZ_TILE16
#define BOLTZ_TILE16 16
#endif
#ifndef BOLTZ_TILE24
#define BOLTZ_TILE24 24
#endif
__host__ __device__ constexpr int conv_tile(int n) {
    return n == 32 ? 16 : n == 24 ? BOLTZ_TILE24 : n == 16 ? BOLTZ_TILE16 : n;
}
#ifndef BOLTZ_CONV_WARPS
#define BOLTZ_CONV_WARPS 4
#endif
#ifndef BOLTZ_TERM_HX
#define BOLTZ_TERM_HX 0  // term arithmetic: 0 = (x*y) then h*, 1 = (h*x) then *y
#endif
// 3 = k_conv_kcs (one kernel per k-chunk, y/H staged), 1 = k_conv_pipe,
// 0 = k_conv; -1 = per-N default
#ifndef BOLTZ_CONV_KERNEL
#define BOLTZ_CONV_KERNEL -1
#endif
#ifndef BOLTZ_KERNEL24
#define BOLTZ_KERNEL24 3
#endif
__host__ __device__ constexpr int conv_kernel_for(int n) {
    return BOLTZ_CONV_KERNEL >= 0 ? BOLTZ_CONV_KERNEL : (n == 32 ? 3 : n == 24 ? BOLTZ_KERNEL24 : 1);
}
constexpr int kConvWarps = BOLTZ_CONV_WARPS;  // cell groups per CTA (share the row stream / H via L1)

// Term arithmetic.  acc += h * x * y for complex x = a + ib (per diagonal),
// y = c + id (per term), real h.  Default: 2 DMUL + 4 DFMA.  Gauss form
// (BOLTZ_TERM_GAUSS): the y window holds (c, c + d, d - c) and the diagonal
// a + b, so that with t = c (a + b)
//   Re = t - b (c + d) = ac - bd,   Im = t + a (d - c) = ad + bc
// costs 1 DMUL + 2 DFMA, and the accumulation 2 DFMA: 5 FP64 instructions
// per term instead of 6 (the sums are paid once per y value and diagonal).
#ifndef BOLTZ_TERM_GAUSS
#define BOLTZ_TERM_GAUSS 0  // every kernel; the per-kernel defaults below win otherwise
#endif
struct YG {
    double c, s, t;  // c, c + d, d - c of y = c + i d
};
__device__ __forceinline__ YG to_yg(double2 v) { return YG{v.x, v.x + v.y, v.y - v.x}; }
#if BOLTZ_TERM_GAUSS
using YElem = YG;
__device__ __forceinline__ YG to_y(double2 v) { return to_yg(v); }
#else
using YElem = double2;
__device__ __forceinline__ double2 to_y(double2 v) { return v; }
#endif
// k_conv_mirror: kk passes of its bands (BOLTZ_MIRROR_KS) and its term form
#ifndef BOLTZ_MIRROR_KS
#define BOLTZ_MIRROR_KS 1
#endif
// B200, cfg2 RK2 step, k_conv_mirror<16> K2 ms: 11.0 (6-instruction term) | 12.0 Gauss,
// KS = 2 | 12.4 Gauss, KS = 4 | 11.3 KS = 2: kept at the 6-instruction term, KS = 1
#ifndef BOLTZ_MIRROR_GAUSS
#define BOLTZ_MIRROR_GAUSS BOLTZ_TERM_GAUSS
#endif
constexpr int kMirrorKS = BOLTZ_MIRROR_KS;

// does diagonal m3 carry a term of tile (kc, sc), type ty, in kk pass q of ks?
__host__ __device__ constexpr bool diag_used_q(int n, int t, int kc, int sc, int m3, int ty, int ks, int q) {
    bool any = false;
    for (int kk = q * t / ks; kk < (q + 1) * t / ks; ++kk) any = any || band_term_t(n, t, kc, sc, m3, kk, ty);
    return any;
}

// one tile of terms: acc[kk] += H * x[m3] * y[j]; the x source and the
// per-diagonal hook (x refill) are policies.  KS > 1 walks the band in KS
// passes over kk ranges (pass, diagonal, kk order -- the table builder lays
// the slab out the same way), so only T / KS accumulators are live at a time
// while x is read KS times per diagonal.
template <int N, int T, int NK, int KC, int TI, int TY = BT_FULL, int KS = 1, typename YT, typename XAt,
          typename AfterDiag>
__device__ __forceinline__ void band_tile(double2 (&acc)[T], const YT (&y)[T], XAt x_at, const double2* hs,
                                          int& p, double2& hb, AfterDiag after) {
    constexpr int SC = band_tile_sc(NK, KC, TI);
    constexpr bool GAUSS = std::is_same<YT, YG>::value;
#pragma unroll
    for (int q = 0; q < KS; ++q)
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const int m3 = band_diag(N, NK, KC, TI, i);
        if (!diag_used_q(N, T, KC, SC, m3, TY, KS, q)) continue;
        const double2 xm = x_at(m3);
        double xab = 0.0;
        if constexpr (GAUSS) xab = xm.x + xm.y;
#pragma unroll
        for (int kk = q * T / KS; kk < (q + 1) * T / KS; ++kk) {
            if (!band_term_t(N, T, KC, SC, m3, kk, TY)) continue;
            const int j = KC * T + kk - m3 + N / 2 - SC * T;  // y chunk slot
            double h;
            if ((p & 1) == 0) { hb = hs[p >> 1]; h = hb.x; }
            else h = hb.y;
            ++p;
            if constexpr (GAUSS) {
                const double t = y[j].c * xab;
                const double tr = fma(-xm.y, y[j].s, t);
                const double ti = fma(xm.x, y[j].t, t);
                acc[kk].x = fma(h, tr, acc[kk].x);
                acc[kk].y = fma(h, ti, acc[kk].y);
                continue;
            } else {
#if BOLTZ_TERM_HX
            // b = h*x (independent of y and acc), then acc += b*y: 2 DMUL + 4 DFMA
            const double bx = h * xm.x, by = h * xm.y;
            acc[kk].x = fma(bx, y[j].x, acc[kk].x);
            acc[kk].x = fma(-by, y[j].y, acc[kk].x);
            acc[kk].y = fma(bx, y[j].y, acc[kk].y);
            acc[kk].y = fma(by, y[j].x, acc[kk].y);
#else
            const double tr = fma(xm.x, y[j].x, -xm.y * y[j].y);
            const double ti = fma(xm.x, y[j].y, xm.y * y[j].x);
            acc[kk].x = fma(h, tr, acc[kk].x);
            acc[kk].y = fma(h, ti, acc[kk].y);
#endif
            }
        }
        after(i, m3);
    }
}


// row_start holds the CSR offsets of the N*N output rows (N*N+1 ints), then two
// processing orders of the rows: longest row list first and the natural order.
// A CTA of column blockIdx.y (a set of cell groups) uses the longest-first order
// when blockIdx.y >= lpt_from: every column for grids of a few waves, the last
// column only for many-wave grids -- so the final wave is made of short rows
// while the earlier columns keep the L2-friendly natural order (neighbouring
// rows share f-hat rows).  The row order does not change any result.
template <int N>
__device__ __forceinline__ int conv_row(const int* __restrict__ row_start, int b, int lpt) {
    return lpt ? __ldg(row_start + N * N + 1 + b) : b;
}

template <int N, int T>
__device__ __forceinline__ void write_row(double2* __restrict__ B, int g, int row, int kc, int lane,
                                          const double2 (&acc)[T]) {
    constexpr int N3 = N * N * N;
    const int k1 = row / N, k2 = row % N;
    double2* Bg = B + ((size_t)g * N3 + (size_t)row * N) * kLanes + lane;
#pragma unroll
    for (int kk = 0; kk < T; ++kk) {
        const int k3 = kc * T + kk;
        const double s = ((k1 + k2 + k3) & 1) ? -1.0 : 1.0;  // inverse transform's input sign s_k
        Bg[(size_t)k3 * kLanes] = make_double2(s * acc[kk].x, s * acc[kk].y);
    }
}

// ---------------------------------------------------------------------------
// k_conv: direct loads, no staging (kept as the plain reference of the order)
// ---------------------------------------------------------------------------
template <int N, int KC>
__device__ __forceinline__ void conv_rows(const double2* __restrict__ Ag, const double* __restrict__ H,
                                          const int2* __restrict__ ent, int e0, int e1,
                                          double2 (&acc)[conv_tile(N)]) {
    constexpr int T = conv_tile(N), NK = N / T;
    constexpr int SLAB_KC = band_slab_kc(N, T);
    for (int e = e0; e < e1; ++e) {
        const int2 en = __ldg(ent + e);
        const double2* X = Ag + (size_t)en.x * kLanes;
        const double2* Y = Ag + (size_t)en.y * kLanes;
        const double2* Hs = reinterpret_cast<const double2*>(H + ((size_t)e * NK + KC) * SLAB_KC);
        int p = 0;
        double2 hb = make_double2(0.0, 0.0);
        auto xat = [&](int m3) { return ldg2(X + (size_t)m3 * kLanes); };
        auto none = [](int, int) {};
        YElem y[T];
#pragma unroll
        for (int j = 0; j < T; ++j) y[j] = to_y(ldg2(Y + (size_t)(band_tile_sc(NK, KC, 0) * T + j) * kLanes));
        band_tile<N, T, NK, KC, 0>(acc, y, xat, Hs, p, hb, none);
        if constexpr (NK == 2) {
#pragma unroll
            for (int j = 0; j < T; ++j) y[j] = to_y(ldg2(Y + (size_t)(band_tile_sc(NK, KC, 1) * T + j) * kLanes));
            band_tile<N, T, NK, KC, 1>(acc, y, xat, Hs, p, hb, none);
        }
    }
}

template <int N>
__global__ void __launch_bounds__(kLanes* kConvWarps, 1)
k_conv(const double2* __restrict__ A, double2* __restrict__ B, const double* __restrict__ H,
       const int2* __restrict__ ent, const int* __restrict__ row_start, int ngroups, int lpt_from) {
    constexpr int T = conv_tile(N), NK = N / T, N3 = N * N * N;
    const int kc = blockIdx.x % NK, row = conv_row<N>(row_start, blockIdx.x / NK, (int)blockIdx.y >= lpt_from);
    const int lane = threadIdx.x & 31;
    const int g = blockIdx.y * kConvWarps + (threadIdx.x >> 5);
    if (g >= ngroups) return;
    const double2* Ag = A + (size_t)g * N3 * kLanes + lane;
    double2 acc[T];
#pragma unroll
    for (int i = 0; i < T; ++i) acc[i] = make_double2(0.0, 0.0);
    const int e0 = __ldg(row_start + row), e1 = __ldg(row_start + row + 1);
    if (kc == 0) conv_rows<N, 0>(Ag, H, ent, e0, e1, acc);
    else if constexpr (NK > 1) conv_rows<N, (NK > 1 ? 1 : 0)>(Ag, H, ent, e0, e1, acc);
    write_row<N, T>(B, g, row, kc, lane, acc);
}

#ifndef BOLTZ_K0_MINB
#define BOLTZ_K0_MINB 1
#endif
#ifndef BOLTZ_PIPE_TMA
#define BOLTZ_PIPE_TMA 1  // row-pair staging by 1D TMA bulk copies + mbarriers (single-tile rows); 0: per-lane cp.async
#endif
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}"
        ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// an entry list read through a 32-entry window, lane j holding entry wb + j:
// the next entry is one shuffle away instead of a dependent L2 load per entry
// (e is warp-uniform)
struct EntWin {
    const int4* ent;
    int e1, wb, lane;
    int4 win;
    __device__ __forceinline__ EntWin(const int4* ent_, int e0, int e1_, int lane_)
        : ent(ent_), e1(e1_), wb(e0), lane(lane_) {
        win = e0 + lane < e1 ? __ldg(ent + e0 + lane) : make_int4(0, 0, 0, 0);
    }
    __device__ __forceinline__ int4 get(int e) {
        if (e - wb >= 32) {
            wb += 32;
            win = wb + lane < e1 ? __ldg(ent + wb + lane) : make_int4(0, 0, 0, 0);
        }
        const int j = e - wb;
        return make_int4(__shfl_sync(0xffffffffu, win.x, j), __shfl_sync(0xffffffffu, win.y, j),
                         __shfl_sync(0xffffffffu, win.z, j), __shfl_sync(0xffffffffu, win.w, j));
    }
    __device__ __forceinline__ int4 first(int e0) { return get(e0); }
    // entry e + 1 when there is one (else `cur`)
    __device__ __forceinline__ int4 next(int e, bool more, int4 cur) { return more ? get(e + 1) : cur; }
};
// the same interface with one entry loaded ahead (no window registers)
struct EntAhead {
    const int4* ent;
    int e1;
    int4 ahead;
    __device__ __forceinline__ EntAhead(const int4* ent_, int e0, int e1_, int) : ent(ent_), e1(e1_) {
        ahead = e0 + 1 < e1 ? __ldg(ent + e0 + 1) : make_int4(0, 0, 0, 0);
    }
    __device__ __forceinline__ int4 first(int e0) { return __ldg(ent + e0); }
    __device__ __forceinline__ int4 next(int e, bool, int4) {
        const int4 nx = ahead;
        if (e + 2 < e1) ahead = __ldg(ent + e + 2);
        return nx;
    }
};
// k_conv_kcsm at N = 32 through an EntWin instead: measured 72.2 against 71.6 ms
// per 1024-cell collide (no gain: its entry loads are not on the critical path)
#ifndef BOLTZ_KCSM_ENTWIN
#define BOLTZ_KCSM_ENTWIN 0
#endif
// the mirror kernels (N <= 16, ~250 terms per entry): the window.  With one
// entry loaded ahead, the compiler copied the loaded value into the loop-carried
// register right after the load, so every entry waited on an L2 round trip
// (ncu source view of k_conv_mirror2<16>: 1.7% of all stall samples on that copy)
#ifndef BOLTZ_MIRROR_ENTWIN
#define BOLTZ_MIRROR_ENTWIN 1
#endif
using EntSrc = std::conditional_t<BOLTZ_MIRROR_ENTWIN != 0, EntWin, EntAhead>;
// 1D TMA: bytes (multiple of 16) global -> this CTA's shared memory, completing on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// Three 1D TMA copies onto one mbarrier (expect_tx of their total) issued by one
// elected lane; called by the whole, converged warp.  Replaces an `if (lane ==
// 0)` block, which ptxas wraps in a divergent ELECT loop per copy (ncu source
// view of k_conv_mirror2<16>: ~2% of all stall samples on that issue code).
#ifndef BOLTZ_TMA_ELECT
#define BOLTZ_TMA_ELECT 1
#endif
// one copy: expect_tx of its bytes + the copy, by one elected lane
__device__ __forceinline__ void bulk_g2s1_elect(unsigned long long* bar, void* d0, const void* s0, unsigned b0) {
    asm volatile(
        "{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n"
        " @p fence.proxy.async.shared::cta;\n"
        " @p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
        " @p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3], %1, [%0];\n}"
        ::"r"(smem_u32(bar)), "r"(b0), "r"(smem_u32(d0)), "l"(s0)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s3_elect(unsigned long long* bar, void* d0, const void* s0, unsigned b0,
                                                void* d1, const void* s1, unsigned b1, void* d2, const void* s2,
                                                unsigned b2) {
    asm volatile(
        "{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n"
        " @p fence.proxy.async.shared::cta;\n"
        " @p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
        " @p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3], %4, [%0];\n"
        " @p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%5], [%6], %7, [%0];\n"
        " @p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%8], [%9], %10, [%0];\n}"
        ::"r"(smem_u32(bar)), "r"(b0 + b1 + b2), "r"(smem_u32(d0)), "l"(s0), "r"(b0), "r"(smem_u32(d1)), "l"(s1),
          "r"(b1), "r"(smem_u32(d2)), "l"(s2), "r"(b2)
        : "memory");
}

// ---------------------------------------------------------------------------
// k_conv_kcs: one k-chunk per kernel; the y row and the H slab of the next row
// pair are staged in shared memory by cp.async while the current one computes
// (H is DRAM-resident at N=32: 1.85 GB), x is read per diagonal from L2.
//   per warp: y[N][32] double2 | H[2][SLAB_KC] double   (N=32: 22.3 KB)
// ---------------------------------------------------------------------------
template <int N>
struct KcsLayout {
    static constexpr int T = conv_tile(N);
    static constexpr int NK = N / T;
    static constexpr int SLAB_KC = band_slab_kc(N, T);
    static constexpr int Y_BYTES = N * kLanes * 16;
    static constexpr int H_BYTES = SLAB_KC * 8;
    static constexpr int WARP_BYTES = Y_BYTES + 2 * H_BYTES + (BOLTZ_PIPE_TMA && NK == 2 ? 16 : 0);  // + 2 mbarriers
};

template <int N, int KC>
__global__ void __launch_bounds__(kLanes* kConvWarps, BOLTZ_K0_MINB)
k_conv_kcs(const double2* __restrict__ A, double2* __restrict__ B, const double* __restrict__ H,
           const int2* __restrict__ ent, const int* __restrict__ row_start, int ngroups, int lpt_from) {
    using LY = KcsLayout<N>;
    constexpr int T = LY::T, NK = LY::NK, N3 = N * N * N;
    extern __shared__ __align__(16) char smem[];
    const int row = conv_row<N>(row_start, blockIdx.x, (int)blockIdx.y >= lpt_from);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int g = blockIdx.y * kConvWarps + wid;
    if (g >= ngroups) return;
    char* wsm = smem + wid * LY::WARP_BYTES;
    double2* ys = reinterpret_cast<double2*>(wsm);
    char* hbase = wsm + LY::Y_BYTES;
    const double2* Ag = A + (size_t)g * N3 * kLanes + lane;
    auto issue_h = [&](int buf, int e) {
        const char* hg = reinterpret_cast<const char*>(H + ((size_t)e * NK + KC) * LY::SLAB_KC);
        for (int o = lane * 16; o < LY::H_BYTES; o += kLanes * 16) cp_async16(hbase + buf * LY::H_BYTES + o, hg + o);
    };
    auto issue_y = [&](int2 en) {
        const double2* Y = Ag + (size_t)en.y * kLanes;
#pragma unroll
        for (int j = 0; j < N; ++j) cp_async16(ys + j * kLanes + lane, Y + (size_t)j * kLanes);
    };
    double2 acc[T];
#pragma unroll
    for (int i = 0; i < T; ++i) acc[i] = make_double2(0.0, 0.0);
    const int e0 = __ldg(row_start + row), e1 = __ldg(row_start + row + 1);
    // 1D TMA staging (N=32; measured neutral-to-negative at N=24): the next
    // entry's H slab (double-buffered) and y row (single buffer, refilled once
    // its chunk is in registers) are two bulk copies by lane 0, each arriving
    // (with its byte count) on the slot's 2-count mbarrier
    constexpr bool KTMA = BOLTZ_PIPE_TMA && NK == 2;
    if constexpr (KTMA) {
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(wsm + LY::Y_BYTES + 2 * LY::H_BYTES);
    const double2* Abase = Ag - lane;
    auto tma_h = [&](int slot, int e) {
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar + slot, LY::H_BYTES);
            bulk_g2s(hbase + slot * LY::H_BYTES, H + ((size_t)e * NK + KC) * LY::SLAB_KC, LY::H_BYTES, bar + slot);
        }
    };
    auto tma_y = [&](int slot, int2 en) {
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar + slot, LY::Y_BYTES);
            bulk_g2s(ys, Abase + (size_t)en.y * kLanes, LY::Y_BYTES, bar + slot);
        }
    };
    if (e0 < e1) {
        if (lane == 0) {
            mbar_init(bar, 2);
            mbar_init(bar + 1, 2);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        int2 en = __ldg(ent + e0);
        int2 en_ahead = e0 + 1 < e1 ? __ldg(ent + e0 + 1) : en;
        tma_y(0, en);
        tma_h(0, e0);
        mbar_wait(bar, 0);
        for (int e = e0; e < e1; ++e) {
            const int i = e - e0, cur = i & 1;
            const bool more = e + 1 < e1;
            const int2 nx = en_ahead;
            if (e + 2 < e1) en_ahead = __ldg(ent + e + 2);
            __syncwarp();  // every lane finished reading H[cur^1]
            if (more) tma_h(cur ^ 1, e + 1);
            const double2* X = Ag + (size_t)en.x * kLanes;
            const double2* hs = reinterpret_cast<const double2*>(hbase + cur * LY::H_BYTES);
            int p = 0;
            double2 hb = make_double2(0.0, 0.0);
            auto xat = [&](int m3) { return ldg2(X + (size_t)m3 * kLanes); };
            auto none = [](int, int) {};
            YElem y[T];
#pragma unroll
            for (int j = 0; j < T; ++j) y[j] = to_y(ys[(band_tile_sc(NK, KC, 0) * T + j) * kLanes + lane]);
            if constexpr (NK == 1) {
                __syncwarp();  // every lane holds its y chunk: the buffer may be refilled
                if (more) tma_y(cur ^ 1, nx);
                band_tile<N, T, NK, KC, 0>(acc, y, xat, hs, p, hb, none);
            } else {
                band_tile<N, T, NK, KC, 0>(acc, y, xat, hs, p, hb, none);
#pragma unroll
                for (int j = 0; j < T; ++j) y[j] = to_y(ys[(band_tile_sc(NK, KC, 1) * T + j) * kLanes + lane]);
                __syncwarp();
                if (more) tma_y(cur ^ 1, nx);
                band_tile<N, T, NK, KC, 1>(acc, y, xat, hs, p, hb, none);
            }
            if (more) mbar_wait(bar + (cur ^ 1), (unsigned)(((i + 1) >> 1) & 1));
            en = nx;
        }
    }
    } else {
    if (e0 < e1) {
        int2 en = __ldg(ent + e0);
        int2 en_ahead = e0 + 1 < e1 ? __ldg(ent + e0 + 1) : en;  // next entry, loaded a row early
        issue_y(en);
        issue_h(0, e0);
        cp_async_commit();
        cp_async_wait_all();
        __syncwarp();
        for (int e = e0; e < e1; ++e) {
            const int cur = (e - e0) & 1;
            const bool more = e + 1 < e1;
            const int2 nx = en_ahead;
            if (e + 2 < e1) en_ahead = __ldg(ent + e + 2);
            __syncwarp();  // every lane finished reading H[cur^1]
            if (more) issue_h(cur ^ 1, e + 1);
            cp_async_commit();
            const double2* X = Ag + (size_t)en.x * kLanes;
            const double2* hs = reinterpret_cast<const double2*>(hbase + cur * LY::H_BYTES);
            int p = 0;
            double2 hb = make_double2(0.0, 0.0);
            auto xat = [&](int m3) { return ldg2(X + (size_t)m3 * kLanes); };
            auto none = [](int, int) {};
            YElem y[T];
#pragma unroll
            for (int j = 0; j < T; ++j) y[j] = to_y(ys[(band_tile_sc(NK, KC, 0) * T + j) * kLanes + lane]);
            if constexpr (NK == 1) {
                if (more) issue_y(nx);  // own-lane slots, just read
                cp_async_commit();
                band_tile<N, T, NK, KC, 0>(acc, y, xat, hs, p, hb, none);
            } else {
                band_tile<N, T, NK, KC, 0>(acc, y, xat, hs, p, hb, none);
#pragma unroll
                for (int j = 0; j < T; ++j) y[j] = to_y(ys[(band_tile_sc(NK, KC, 1) * T + j) * kLanes + lane]);
                if (more) issue_y(nx);
                cp_async_commit();
                band_tile<N, T, NK, KC, 1>(acc, y, xat, hs, p, hb, none);
            }
            if (more) {
                cp_async_wait_all();
                __syncwarp();
            }
            en = nx;
        }
    }
    }
    write_row<N, T>(B, g, row, KC, lane, acc);
}

// ---------------------------------------------------------------------------
// k_conv_pipe: x double-buffered, full y row staged, H double-buffered
//   per warp: x[2][N][32] + y[N][32] double2, H[2][SLAB_KC] double
// ---------------------------------------------------------------------------
template <int N>
struct PipeLayout {
    static constexpr int T = conv_tile(N);
    static constexpr int NK = N / T;
    static constexpr int SLAB_KC = band_slab_kc(N, T);
    static constexpr int X_BYTES = N * kLanes * 16;
    static constexpr int H_BYTES = SLAB_KC * 8;
    static constexpr bool TMA = BOLTZ_PIPE_TMA && NK == 1;
    static constexpr int WARP_BYTES = 3 * X_BYTES + 2 * H_BYTES + (TMA ? 16 : 0);  // + 2 mbarriers
};

template <int N, int KC>
__device__ __forceinline__ void pipe_rows(char* wsm, const double2* __restrict__ Ag, const double* __restrict__ H,
                                          const int2* __restrict__ ent, int e0, int e1, int lane,
                                          double2 (&acc)[conv_tile(N)]) {
    using PL = PipeLayout<N>;
    constexpr int T = PL::T, NK = PL::NK;
    const double2* ys = reinterpret_cast<const double2*>(wsm + 2 * PL::X_BYTES);
    if constexpr (PL::TMA) {
        // the next row pair's x row (8 KB at N=16, contiguous in the group layout),
        // y row and H slab: three bulk copies issued by lane 0, completing on the
        // slot's mbarrier (slot = entry parity); every lane waits on the parity
        unsigned long long* bar = reinterpret_cast<unsigned long long*>(wsm + 3 * PL::X_BYTES + 2 * PL::H_BYTES);
        const double2* Abase = Ag - lane;
        auto issue = [&](int slot, int2 en, int e) {  // the whole warp (converged)
            if constexpr (BOLTZ_TMA_ELECT) {
                bulk_g2s3_elect(bar + slot, wsm + slot * PL::X_BYTES, Abase + (size_t)en.x * kLanes, PL::X_BYTES,
                                wsm + 2 * PL::X_BYTES, Abase + (size_t)en.y * kLanes, PL::X_BYTES,
                                wsm + 3 * PL::X_BYTES + slot * PL::H_BYTES, H + (size_t)e * PL::SLAB_KC, PL::H_BYTES);
            } else if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads of the slot are done
                mbar_expect_tx(bar + slot, 2 * PL::X_BYTES + PL::H_BYTES);
                bulk_g2s(wsm + slot * PL::X_BYTES, Abase + (size_t)en.x * kLanes, PL::X_BYTES, bar + slot);
                bulk_g2s(wsm + 2 * PL::X_BYTES, Abase + (size_t)en.y * kLanes, PL::X_BYTES, bar + slot);
                bulk_g2s(wsm + 3 * PL::X_BYTES + slot * PL::H_BYTES, H + (size_t)e * PL::SLAB_KC, PL::H_BYTES,
                         bar + slot);
            }
        };
        if (e0 >= e1) return;
        if (lane == 0) {
            mbar_init(bar, 1);
            mbar_init(bar + 1, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        int2 en_next = __ldg(ent + e0);
        int2 en_ahead = e0 + 1 < e1 ? __ldg(ent + e0 + 1) : en_next;
        issue(0, en_next, e0);
        mbar_wait(bar, 0);
        YElem y[T];
#pragma unroll
        for (int j = 0; j < T; ++j) y[j] = to_y(ys[j * kLanes + lane]);
        for (int e = e0; e < e1; ++e) {
            const int i = e - e0, cur = i & 1;
            const bool more = e + 1 < e1;
            en_next = en_ahead;
            if (e + 2 < e1) en_ahead = __ldg(ent + e + 2);
            __syncwarp();  // every lane read y (registers) and is done with slot cur^1
            if (more) issue(cur ^ 1, en_next, e + 1);
            const double2* xs = reinterpret_cast<const double2*>(wsm + cur * PL::X_BYTES);
            const double2* hs = reinterpret_cast<const double2*>(wsm + 3 * PL::X_BYTES + cur * PL::H_BYTES);
            int p = 0;
            double2 hb = make_double2(0.0, 0.0);
            auto xat = [&](int m3) { return xs[m3 * kLanes + lane]; };
            auto none = [](int, int) {};
            band_tile<N, T, NK, KC, 0>(acc, y, xat, hs, p, hb, none);
            if (more) {
                mbar_wait(bar + (cur ^ 1), (unsigned)(((i + 1) >> 1) & 1));
#pragma unroll
                for (int j = 0; j < T; ++j) y[j] = to_y(ys[j * kLanes + lane]);
            }
        }
        return;
    }
    auto issue_xh = [&](int buf, int2 en, int e) {
        double2* xs = reinterpret_cast<double2*>(wsm + buf * PL::X_BYTES);
        const double2* X = Ag + (size_t)en.x * kLanes;
#pragma unroll
        for (int j = 0; j < N; ++j) cp_async16(xs + j * kLanes + lane, X + (size_t)j * kLanes);
        char* hs = wsm + 3 * PL::X_BYTES + buf * PL::H_BYTES;
        const char* hg = reinterpret_cast<const char*>(H + ((size_t)e * NK + KC) * PL::SLAB_KC);
        for (int o = lane * 16; o < PL::H_BYTES; o += kLanes * 16) cp_async16(hs + o, hg + o);
        cp_async_commit();
    };
    auto issue_y = [&](int2 en) {
        double2* yw = reinterpret_cast<double2*>(wsm + 2 * PL::X_BYTES);
        const double2* Y = Ag + (size_t)en.y * kLanes;
#pragma unroll
        for (int j = 0; j < N; ++j) cp_async16(yw + j * kLanes + lane, Y + (size_t)j * kLanes);
        cp_async_commit();
    };
    if (e0 >= e1) return;
    int2 en_next = __ldg(ent + e0);
    // the entry two row pairs ahead is loaded one row early, so the cp.async
    // addresses at a row start never wait on a dependent global load
    int2 en_ahead = e0 + 1 < e1 ? __ldg(ent + e0 + 1) : en_next;
    issue_xh(0, en_next, e0);
    issue_y(en_next);
    cp_async_wait_all();
    __syncwarp();
    YElem y[T];
#pragma unroll
    for (int j = 0; j < T; ++j) y[j] = to_y(ys[(band_tile_sc(NK, KC, 0) * T + j) * kLanes + lane]);
    for (int e = e0; e < e1; ++e) {
        const int cur = (e - e0) & 1;
        const bool more = e + 1 < e1;
        en_next = en_ahead;
        if (e + 2 < e1) en_ahead = __ldg(ent + e + 2);
        __syncwarp();
        if (more) issue_xh(cur ^ 1, en_next, e + 1);
        if (NK == 1 && more) issue_y(en_next);
        const double2* xs = reinterpret_cast<const double2*>(wsm + cur * PL::X_BYTES);
        const double2* hs = reinterpret_cast<const double2*>(wsm + 3 * PL::X_BYTES + cur * PL::H_BYTES);
        int p = 0;
        double2 hb = make_double2(0.0, 0.0);
        auto xat = [&](int m3) { return xs[m3 * kLanes + lane]; };
        auto none = [](int, int) {};
        band_tile<N, T, NK, KC, 0>(acc, y, xat, hs, p, hb, none);
        if constexpr (NK == 2) {
#pragma unroll
            for (int j = 0; j < T; ++j) y[j] = to_y(ys[(band_tile_sc(NK, KC, 1) * T + j) * kLanes + lane]);
            if (more) issue_y(en_next);
            band_tile<N, T, NK, KC, 1>(acc, y, xat, hs, p, hb, none);
        }
        if (more) {
            cp_async_wait_all();
            __syncwarp();
#pragma unroll
            for (int j = 0; j < T; ++j) y[j] = to_y(ys[(band_tile_sc(NK, KC, 0) * T + j) * kLanes + lane]);
        }
    }
}

#ifndef BOLTZ_PIPE_MINB
#define BOLTZ_PIPE_MINB 1
#endif
template <int N>
__global__ void __launch_bounds__(kLanes* kConvWarps, BOLTZ_PIPE_MINB)
k_conv_pipe(const double2* __restrict__ A, double2* __restrict__ B, const double* __restrict__ H,
            const int2* __restrict__ ent, const int* __restrict__ row_start, int ngroups, int lpt_from) {
    using PL = PipeLayout<N>;
    constexpr int T = PL::T, NK = PL::NK, N3 = N * N * N;
    extern __shared__ __align__(16) char smem[];
    const int kc = blockIdx.x % NK, row = conv_row<N>(row_start, blockIdx.x / NK, (int)blockIdx.y >= lpt_from);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int g = blockIdx.y * kConvWarps + wid;
    if (g >= ngroups) return;
    char* wsm = smem + wid * PL::WARP_BYTES;
    const double2* Ag = A + (size_t)g * N3 * kLanes + lane;
    double2 acc[T];
#pragma unroll
    for (int i = 0; i < T; ++i) acc[i] = make_double2(0.0, 0.0);
    const int e0 = __ldg(row_start + row), e1 = __ldg(row_start + row + 1);
    if (kc == 0) pipe_rows<N, 0>(wsm, Ag, H, ent, e0, e1, lane, acc);
    else if constexpr (NK > 1) pipe_rows<N, (NK > 1 ? 1 : 0)>(wsm, Ag, H, ent, e0, e1, lane, acc);
    write_row<N, T>(B, g, row, kc, lane, acc);
}

// ---------------------------------------------------------------------------
// Latency schedule (boltz_set_schedule(ctx, 1)) for small batches: a CTA owns
// one (output row, group) and its kConvWarps warps take kConvWarps fixed,
// contiguous segments of the row's entry list -- kConvWarps x the warps of the
// throughput schedule when there are only a few groups, and each warp's list
// is a quarter as long.  Segment partials go to scratch P[s][g][row][k3][lane]
// and k_conv_seg_reduce adds them in segment order.  The per-cell arithmetic
// depends only on the row lists, so results are bitwise independent of batch
// size and composition in this schedule too (they differ from the throughput
// schedule's by round-off: a different summation order).
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int seg_begin(int e0, int e1, int s, int S) {
    return e0 + (int)(((long long)(e1 - e0) * s) / S);
}

// grid = (N^2 rows, groups, S / kConvWarps); warp w of CTA z takes segment
// z * kConvWarps + w of S
template <int N>
__global__ void __launch_bounds__(kLanes* kConvWarps, 1)
k_conv_seg(const double2* __restrict__ A, double2* __restrict__ P, const double* __restrict__ H,
           const int2* __restrict__ ent, const int* __restrict__ row_start, int ngroups, int S) {
    using PL = PipeLayout<N>;
    static_assert(PL::NK == 1, "latency schedule: single-tile rows");
    constexpr int T = PL::T, N3 = N * N * N;
    extern __shared__ __align__(16) char smem[];
    const int row = conv_row<N>(row_start, blockIdx.x, 1);
    const int g = blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int sgm = blockIdx.z * kConvWarps + w;
    char* wsm = smem + w * PL::WARP_BYTES;
    const double2* Ag = A + (size_t)g * N3 * kLanes + lane;
    double2 acc[T];
#pragma unroll
    for (int i = 0; i < T; ++i) acc[i] = make_double2(0.0, 0.0);
    const int e0 = __ldg(row_start + row), e1 = __ldg(row_start + row + 1);
    pipe_rows<N, 0>(wsm, Ag, H, ent, seg_begin(e0, e1, sgm, S), seg_begin(e0, e1, sgm + 1, S), lane, acc);
    double2* Pg = P + (((size_t)sgm * ngroups + g) * N3 + (size_t)row * N) * kLanes + lane;
#pragma unroll
    for (int kk = 0; kk < T; ++kk) Pg[(size_t)kk * kLanes] = acc[kk];
}

// B = s_k * (((0 + P_0) + P_1) + ...) over the S segments
template <int N>
__global__ void __launch_bounds__(256)
k_conv_seg_reduce(const double2* __restrict__ P, double2* __restrict__ B, long long ngroups, int S) {
    constexpr int N3 = N * N * N;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // over ngroups * N3 * kLanes
    const long long total = ngroups * N3 * kLanes;
    if (i >= total) return;
    double2 sum = make_double2(0.0, 0.0);
    for (int sgm = 0; sgm < S; ++sgm) {
        const double2 v = P[(size_t)sgm * total + i];
        sum.x += v.x;
        sum.y += v.y;
    }
    const int idx = (int)((i / kLanes) % N3);
    const int k1 = idx / (N * N), k2 = (idx / N) % N, k3 = idx % N;
    const double sg = ((k1 + k2 + k3) & 1) ? -1.0 : 1.0;  // inverse transform's input sign s_k
    B[i] = make_double2(sg * sum.x, sg * sum.y);
}

// ---------------------------------------------------------------------------
// Cell schedule (boltz_set_schedule(ctx, 5)) for one or a few cells, N <= 16:
// lane = output k3 instead of lane = cell, so a single cell (cfg1) keeps every
// lane busy.  A CTA owns one (output row, cell); the cell's f-hat cube is
// staged in shared memory; warp w's lane slot q (32 / N slots of N lanes)
// walks entries e0 + (w * P + q) + j * (8 * P) of the row's plain-table list
// and, per diagonal m3, adds the term (k3 = lane, m3) when it is in the band:
//   h = H[e][doff(m3) + k3 - klo(m3)]  (consecutive lanes, consecutive h),
//   x = fhat(row m, m3) (smem broadcast), y = fhat(row s, k3 - m3 + N/2).
// The slot partials are then added in a fixed (warp, slot) order, so results
// are bitwise reproducible and independent of the batch; they differ from the
// other schedules by round-off (another summation order).
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int cell_klo(int n, int m3) { return m3 - n / 2 > 0 ? m3 - n / 2 : 0; }
__host__ __device__ constexpr int cell_khi(int n, int m3) { return m3 + n / 2 < n ? m3 + n / 2 : n; }
// slab offset of diagonal m3 in a single-tile plain slab (layout_terms_plain order)
__host__ __device__ constexpr int cell_doff(int n, int m3) {
    int o = 0;
    for (int i = 0; i < m3; ++i) o += cell_khi(n, i) - cell_klo(n, i);
    return o;
}
// warps per (row, cell) CTA; B200, cfg1 (50 RK2 steps as graph replays, two
// runs): 4 warps 2.87 / 2.89 ms, 8: 3.33 / 3.34, 16: 2.98 / 2.98 (16 with 64
// registers: 3.07 / 3.08)
#ifndef BOLTZ_CELL_WARPS
#define BOLTZ_CELL_WARPS 4
#endif
constexpr int kCellWarps = BOLTZ_CELL_WARPS;
template <int N>
struct CellLayout {
    static constexpr int P = kLanes / N;  // entry slots per warp
    static constexpr int N3 = N * N * N;
    static constexpr int CUBE_BYTES = N3 * 16;
    static constexpr int RED_BYTES = kCellWarps * P * N * 16;
    static constexpr int BYTES = CUBE_BYTES + RED_BYTES;
};

// the cells' f-hat cubes, group layout -> contiguous [cell][N^3] (k_conv_cell's input)
template <int N>
__global__ void __launch_bounds__(256) k_cell_gather(const double2* __restrict__ A, double2* __restrict__ C, int ncells) {
    constexpr int N3 = N * N * N;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)ncells * N3) return;
    const int cell = (int)(i / N3), idx = (int)(i % N3);
    C[i] = ldg2(A + ((size_t)(cell / kLanes) * N3 + idx) * kLanes + cell % kLanes);
}

#ifndef BOLTZ_CELL_MINB
#define BOLTZ_CELL_MINB 1
#endif
template <int N>
__global__ void __launch_bounds__(kLanes* kCellWarps, BOLTZ_CELL_MINB)
k_conv_cell(const double2* __restrict__ Cc, double2* __restrict__ B, const double* __restrict__ H,
            const int2* __restrict__ ent, const int* __restrict__ row_start, int slab) {
    using CL = CellLayout<N>;
    constexpr int P = CL::P, N3 = CL::N3, S = kCellWarps * P;
    static_assert(conv_tile(N) == N, "cell schedule: single-tile rows");
    extern __shared__ __align__(16) char smem[];
    double2* cube = reinterpret_cast<double2*>(smem);
    double2* red = reinterpret_cast<double2*>(smem + CL::CUBE_BYTES);
    const int row = blockIdx.x, cell = blockIdx.y;
    const int g = cell / kLanes, cl = cell % kLanes;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int q = lane / N, k3 = lane % N;
    const int e0 = __ldg(row_start + row), e1 = __ldg(row_start + row + 1);
    // this slot's first two entries, loaded before the cube arrives
    const int ea = e0 + w * P + q, eb = ea + S;
    const int2 ena = (q < P && ea < e1) ? __ldg(ent + ea) : make_int2(0, 0);
    const int2 enb = (q < P && eb < e1) ? __ldg(ent + eb) : make_int2(0, 0);
    const double2* Cg = Cc + (size_t)cell * N3;
    for (int i = threadIdx.x; i < N3; i += kLanes * kCellWarps) cube[i] = ldg2(Cg + i);
    __syncthreads();
    double2 acc = make_double2(0.0, 0.0);
    // h of one entry for this lane: every diagonal's load issued up front
    // (unconditional, clamped into the slab; out-of-band terms are skipped)
    auto load_h = [&](int e, double (&hv)[N]) {
        const double* hs = H + (size_t)e * slab;
#pragma unroll
        for (int m3 = 0; m3 < N; ++m3) {
            constexpr int dummy = 0;
            const int lo = cell_klo(N, m3), hi = cell_khi(N, m3);
            const int o = cell_doff(N, m3) + (k3 < lo ? 0 : k3 >= hi ? hi - 1 - lo : k3 - lo) + dummy;
            hv[m3] = __ldg(hs + o);
        }
    };
    auto terms = [&](int2 en, const double (&hv)[N]) {
        const double2* xs = cube + en.x;
        const double2* ys = cube + en.y;
#pragma unroll
        for (int m3 = 0; m3 < N; ++m3) {
            if (k3 < cell_klo(N, m3) || k3 >= cell_khi(N, m3)) continue;
            const double2 xm = xs[m3];
            const double2 yv = ys[k3 - m3 + N / 2];
            const double tr = fma(xm.x, yv.x, -xm.y * yv.y);
            const double ti = fma(xm.x, yv.y, xm.y * yv.x);
            acc.x = fma(hv[m3], tr, acc.x);
            acc.y = fma(hv[m3], ti, acc.y);
        }
    };
    if (q < P) {
        // two entries per step: 2N loads of h in flight per lane
        int e = ea;
        int2 en0 = ena, en1 = enb;
        for (; e + S < e1; e += 2 * S) {
            double h0[N], h1[N];
            load_h(e, h0);
            load_h(e + S, h1);
            const int2 nx0 = e + 2 * S < e1 ? __ldg(ent + e + 2 * S) : en0;
            const int2 nx1 = e + 3 * S < e1 ? __ldg(ent + e + 3 * S) : en1;
            terms(en0, h0);
            terms(en1, h1);
            en0 = nx0;
            en1 = nx1;
        }
        if (e < e1) {
            double h0[N];
            load_h(e, h0);
            terms(en0, h0);
        }
        red[(w * P + q) * N + k3] = acc;
    }
    __syncthreads();
    if (threadIdx.x < N) {
        double2 sum = make_double2(0.0, 0.0);
        for (int i = 0; i < S; ++i) {
            const double2 v = red[i * N + threadIdx.x];
            sum.x += v.x;
            sum.y += v.y;
        }
        const int k1 = row / N, k2 = row % N, kk = threadIdx.x;
        const double sg = ((k1 + k2 + kk) & 1) ? -1.0 : 1.0;  // inverse transform's input sign s_k
        B[((size_t)g * N3 + (size_t)row * N + kk) * kLanes + cl] = make_double2(sg * sum.x, sg * sum.y);
    }
}

// ---------------------------------------------------------------------------
// k_conv_mirror (single-tile rows, TMA staging): the Hermitian mirror schedule.
// A work item is an output row r with no mirror partner (k1 = 0, k2 = 0 or
// r = N - r), or a pair (r, r' = N - r).  Its entries are one contiguous list
//     [A(r) | FULL(r) | REST(r) | FULL(r') | REST(r')]
// (int4 {x row, y row, H offset, band type}), staged by one continuous TMA
// pipeline.  One warp (one 32-cell group) runs the item:
//   after A(r):   acc holds the interior sums of r; conj(acc[N - k3']) goes to
//                 row r' of B (k3' = 1..N-1, 0 at k3' = 0); r keeps summing
//   after B(r):   row r is written; acc reloads row r' of B
//   at the end:   row r' (or r for a single row) is written
// The warp owns both rows, so the order is fixed and no other warp touches
// them.  Only for collide / RK2, whose fhat is the transform of a real f.
// item[] = {r, r' (-1: none), begin, end of A, begin of r', end}.
// ---------------------------------------------------------------------------
constexpr int kItemInts = 6;

// A CTA's (item or row-list index, cell-group column).  Columns below lpt_from
// take the items longest-first (head_lpt: blockIdx.x indexes `order`) or in
// their natural, L2-friendly order (k_conv_kcsm / k_conv_kcsr); the last
// gridDim.y - lpt_from columns are scheduled jointly: their CTAs walk the items
// longest-first with the columns innermost, so the final waves hold the
// shortest items of every tail column (a list schedule closer to LPT over the
// whole tail; the tail columns' f-hat stays L2-resident).  lpt_from >= gridDim.y:
// every column longest-first.  The assignment does not change any result.
__device__ __forceinline__ int2 lpt_unit(const int* __restrict__ order, int lpt_from, bool head_lpt) {
    if ((int)blockIdx.y < lpt_from) return make_int2(head_lpt ? __ldg(order + blockIdx.x) : (int)blockIdx.x, (int)blockIdx.y);
    const int k = (int)gridDim.y - lpt_from;
    const int u = ((int)blockIdx.y - lpt_from) * (int)gridDim.x + (int)blockIdx.x;
    return make_int2(__ldg(order + u / k), lpt_from + u % k);
}
__device__ __forceinline__ int2 mirror_unit(const int* __restrict__ order, int lpt_from) {
    return lpt_unit(order, lpt_from, true);
}

template <int N>
struct MirrorLayout {
    static constexpr int X_BYTES = N * kLanes * 16;
    static constexpr int H_BYTES = mirror_slab(N, BT_FULL) * 8;
    static constexpr int WARP_BYTES = 3 * X_BYTES + 2 * H_BYTES + 16;  // + 2 mbarriers
};

template <int N>
__global__ void __launch_bounds__(kLanes* kConvWarps, 1)
k_conv_mirror(const double2* __restrict__ A, double2* __restrict__ B, const double* __restrict__ H,
              const int4* __restrict__ ent, const int* __restrict__ items, const int* __restrict__ order, int ngroups,
              int lpt_from) {
    using PL = MirrorLayout<N>;
    static_assert(PipeLayout<N>::TMA, "the mirror schedule runs on the TMA pipe (single-tile rows)");
    constexpr int T = N, N3 = N * N * N;
    extern __shared__ __align__(16) char smem[];
    const int2 unit = mirror_unit(order, lpt_from);
    const int* it = items + kItemInts * unit.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int g = unit.y * kConvWarps + wid;
    if (g >= ngroups) return;
    const int r = __ldg(it), rm = __ldg(it + 1);
    const int e_begin = __ldg(it + 2), e_endA = __ldg(it + 3), e_rm = __ldg(it + 4), e_end = __ldg(it + 5);
    char* wsm = smem + wid * PL::WARP_BYTES;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(wsm + 3 * PL::X_BYTES + 2 * PL::H_BYTES);
    const double2* ys = reinterpret_cast<const double2*>(wsm + 2 * PL::X_BYTES);
    const double2* Abase = A + (size_t)g * N3 * kLanes;
    double2* Bm = B + ((size_t)g * N3 + (size_t)(rm < 0 ? 0 : rm) * N) * kLanes + lane;
    auto issue = [&](int slot, int4 en) {
        if (lane == 0) {
            const unsigned hb = 8u * (en.w == BT_A ? mirror_slab(N, BT_A) : en.w == BT_REST ? mirror_slab(N, BT_REST)
                                                                                         : mirror_slab(N, BT_FULL));
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar + slot, 2 * PL::X_BYTES + hb);
            bulk_g2s(wsm + slot * PL::X_BYTES, Abase + (size_t)en.x * kLanes, PL::X_BYTES, bar + slot);
            bulk_g2s(wsm + 2 * PL::X_BYTES, Abase + (size_t)en.y * kLanes, PL::X_BYTES, bar + slot);
            bulk_g2s(wsm + 3 * PL::X_BYTES + slot * PL::H_BYTES, H + (size_t)(unsigned)en.z, hb, bar + slot);
        }
    };
    double2 acc[T];
#pragma unroll
    for (int i = 0; i < T; ++i) acc[i] = make_double2(0.0, 0.0);
    // the item's segment boundaries (r' parts only for pairs)
    auto boundary = [&](int e) {
        if (rm < 0) return;
        if (e == e_endA) {  // A(r) done: its conjugate, k3-reversed, seeds row r' (row r keeps summing)
            Bm[0] = make_double2(0.0, 0.0);
#pragma unroll
            for (int k = 1; k < N; ++k) Bm[(size_t)k * kLanes] = make_double2(acc[N - k].x, -acc[N - k].y);
        }
        if (e == e_rm) {  // row r complete: write it, continue with row r'
            write_row<N, T>(B, g, r, 0, lane, acc);
#pragma unroll
            for (int k = 0; k < N; ++k) acc[k] = Bm[(size_t)k * kLanes];
        }
    };
    if (e_begin < e_end) {
        if (lane == 0) {
            mbar_init(bar, 1);
            mbar_init(bar + 1, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        EntSrc src(ent, e_begin, e_end, lane);
        int4 en = src.first(e_begin);
        issue(0, en);
        mbar_wait(bar, 0);
        using YM = std::conditional_t<BOLTZ_MIRROR_GAUSS != 0, YG, double2>;
        auto to_ym = [](double2 v) {
            if constexpr (BOLTZ_MIRROR_GAUSS != 0) return to_yg(v);
            else return v;
        };
        YM y[T];
#pragma unroll
        for (int j = 0; j < T; ++j) y[j] = to_ym(ys[j * kLanes + lane]);
        for (int e = e_begin; e < e_end; ++e) {
            const int i = e - e_begin, cur = i & 1;
            const bool more = e + 1 < e_end;
            const int4 nx = src.next(e, more, en);
            boundary(e);
            __syncwarp();  // every lane read y (registers) and is done with slot cur^1
            if (more) issue(cur ^ 1, nx);
            const double2* xs = reinterpret_cast<const double2*>(wsm + cur * PL::X_BYTES);
            const double2* hs = reinterpret_cast<const double2*>(wsm + 3 * PL::X_BYTES + cur * PL::H_BYTES);
            auto xat = [&](int m3) { return xs[m3 * kLanes + lane]; };
            auto none = [](int, int) {};
            double2 hb = make_double2(0.0, 0.0);
            if (en.w != BT_REST) {  // warp-uniform: A, or the A half of a FULL entry
                int p = 0;
                band_tile<N, T, 1, 0, 0, BT_A, kMirrorKS>(acc, y, xat, hs, p, hb, none);
            }
            if (en.w != BT_A) {  // REST, or the REST half of a FULL entry
                int p = 0;
                band_tile<N, T, 1, 0, 0, BT_REST, kMirrorKS>(acc, y, xat, hs + (en.w == BT_FULL ? mirror_slab(N, BT_A) / 2 : 0),
                                                  p, hb, none);
            }
            if (more) {
                mbar_wait(bar + (cur ^ 1), (unsigned)(((i + 1) >> 1) & 1));
#pragma unroll
                for (int j = 0; j < T; ++j) y[j] = to_ym(ys[j * kLanes + lane]);
            }
            en = nx;
        }
    }
    boundary(e_end);  // boundaries that coincide with the end of the list
    write_row<N, T>(B, g, rm >= 0 ? rm : r, 0, lane, acc);
}

// ---------------------------------------------------------------------------
// k_conv_mirror2 (single-tile rows, TMA staging, TMEM): the mirror schedule
// with every interior input row staged once.  k_conv_mirror stages an interior
// row three times -- A(r), REST(r), REST(r') -- because its only accumulator
// is the register row of the output being summed.  Here an entry of an
// interior input row (type BT_A below: "I") runs
//   A     (diagonal-major band, registers)      -> acc        (row r)
//   REST  (k3-major, 4 outputs per TMEM access) -> T_r  (TMEM, row r)
//   REST' (k3-major)                             -> T_r' (TMEM, row r')
// REST' is r' = N - r's own non-mirrored terms, computed from r's staged rows:
// for real f, fhat(N - m) = conj fhat(m) per axis, so x'[m3'] = conj x[N - m3']
// (m3' >= 1) and x'[0] = fhat(N - m1, N - m2, 0), one extra value per row
// (likewise y'); its weights are r''s own (k_build_H: term.x >= kMirrorTermFlag).
// A FULL entry (non-interior input rows; all rows of an unpaired output row)
// runs the A and the REST band (diagonal-major) into acc.
//   after the I entries: conj(acc[N - k3']) seeds row r' of B (k3' >= 1)
//   after FULL(r):       acc += T_r, row r written; acc = B row r'
//   at the end:          acc += T_r' (T_r for an unpaired row), row written
// Slabs (doubles, even-padded pieces): FULL [A band | REST band],
// I [A band | REST k3-major | REST' k3-major].  Items as k_conv_mirror:
// {r, r' (-1), begin, end of I, begin of r', end}.
// TMEM: each CTA allocates 2 x 4N 32-bit columns per lane (N <= 16: 128);
// warp w uses lanes 32 (w % 4) .. +31; T_r at column 0, T_r' at 4N.
// ---------------------------------------------------------------------------
constexpr int kMirrorTermFlag = 64;  // term.x >= 64: a REST' term, k3' = x - 64, weights of q' = N - q
__host__ __device__ inline int4 mirror_q(int n, int4 q) { return make_int4(n - q.x, n - q.y, n - q.z, n - q.w); }

__host__ __device__ constexpr bool single_band(int n, int k3, int m3) {
    const int s3 = k3 - m3 + n / 2;
    return s3 >= 0 && s3 < n;
}
__host__ __device__ constexpr bool rest_term(int n, int k3, int m3) {
    return single_band(n, k3, m3) && type_term(n, BT_REST, k3, m3);
}
__host__ __device__ constexpr int rest_terms(int n) {
    int c = 0;
    for (int k3 = 0; k3 < n; ++k3)
        for (int m3 = 0; m3 < n; ++m3) c += rest_term(n, k3, m3) ? 1 : 0;
    return c;
}
// slab pieces of k_conv_mirror2 (doubles)
__host__ __device__ constexpr int m2_a(int n) { return band_slab_type(n, BT_A); }
__host__ __device__ constexpr int m2_r(int n) { return (rest_terms(n) + 1) & ~1; }
__host__ __device__ constexpr int m2_slab(int n, int ty) { return ty == BT_A ? m2_a(n) + 2 * m2_r(n) : m2_a(n) + m2_r(n); }
__host__ __device__ constexpr int m2_tmem_cols(int n) { return 8 * n <= 32 ? 32 : 8 * n <= 64 ? 64 : 8 * n <= 128 ? 128 : 256; }

template <int N>
struct Mirror2Layout {
    static constexpr int X_BYTES = N * kLanes * 16;
    static constexpr int H_BYTES = m2_slab(N, BT_A) * 8;
    static constexpr int WARP_BYTES = 3 * X_BYTES + 2 * H_BYTES + 16;  // + 2 mbarriers
    static constexpr int CTA_BYTES = kConvWarps * WARP_BYTES + 16;     // + the TMEM base address
};

// TMEM <-> registers, 4 complex values (16 columns) of this thread's lane
__device__ __forceinline__ void tm_ld4c(uint32_t ta, double2 (&v)[4]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(ta));
#pragma unroll
    for (int i = 0; i < 4; ++i)
        v[i] = make_double2(__hiloint2double(r[4 * i + 1], r[4 * i]), __hiloint2double(r[4 * i + 3], r[4 * i + 2]));
}
__device__ __forceinline__ void tm_st4c(uint32_t ta, const double2 (&v)[4]) {
    uint32_t r[16];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        r[4 * i] = (uint32_t)__double2loint(v[i].x);
        r[4 * i + 1] = (uint32_t)__double2hiint(v[i].x);
        r[4 * i + 2] = (uint32_t)__double2loint(v[i].y);
        r[4 * i + 3] = (uint32_t)__double2hiint(v[i].y);
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(ta), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
          "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
}

// stores complete before TMEM is read again (tm_st4c does not wait)
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// one term of a REST pass into a (PRIME: REST' of the partner row)
template <int N, bool PRIME, int K3, int M3>
__device__ __forceinline__ void m2_term(double2& a, double h, const double2 (&y)[N], const double2* __restrict__ xs,
                                        int lane, double2 X0, double2 Y0) {
    constexpr int S3 = K3 - M3 + N / 2;
    if constexpr (!PRIME) {
        const double2 xm = xs[M3 * kLanes + lane];
        const double tr = fma(xm.x, y[S3].x, -xm.y * y[S3].y);
        const double ti = fma(xm.x, y[S3].y, xm.y * y[S3].x);
        a.x = fma(h, tr, a.x);
        a.y = fma(h, ti, a.y);
    } else if constexpr (M3 == 0) {  // X0 * conj(y[N - s3])  (s3 >= 1 here)
        const double2 yv = y[(N - S3) % N];
        const double tr = fma(X0.x, yv.x, X0.y * yv.y);
        const double ti = fma(X0.y, yv.x, -X0.x * yv.y);
        a.x = fma(h, tr, a.x);
        a.y = fma(h, ti, a.y);
    } else if constexpr (S3 == 0) {  // conj(x[N - m3]) * Y0
        const double2 xm = xs[(N - M3) * kLanes + lane];
        const double tr = fma(xm.x, Y0.x, xm.y * Y0.y);
        const double ti = fma(xm.x, Y0.y, -xm.y * Y0.x);
        a.x = fma(h, tr, a.x);
        a.y = fma(h, ti, a.y);
    } else {  // conj(x[N - m3] * y[N - s3])
        const double2 xm = xs[(N - M3) * kLanes + lane];
        const double2 yv = y[(N - S3) % N];
        const double tr = fma(xm.x, yv.x, -xm.y * yv.y);
        const double ti = fma(xm.x, yv.y, xm.y * yv.x);
        a.x = fma(h, tr, a.x);
        a.y = fma(-h, ti, a.y);
    }
}

// the REST terms of outputs k3 = 4B .. 4B+3 into a[4]; p / hb: the slab cursor
template <int N, bool PRIME, int B, int Q = 0, int M3 = 0>
__device__ __forceinline__ void m2_batch(double2 (&a)[4], const double2 (&y)[N], const double2* __restrict__ xs,
                                         int lane, const double2* __restrict__ hs, int& p, double2& hb, double2 X0,
                                         double2 Y0) {
    if constexpr (Q < 4) {
        if constexpr (M3 < N) {
            if constexpr (rest_term(N, 4 * B + Q, M3)) {
                double h;
                if ((p & 1) == 0) { hb = hs[p >> 1]; h = hb.x; }
                else h = hb.y;
                ++p;
                m2_term<N, PRIME, 4 * B + Q, M3>(a[Q], h, y, xs, lane, X0, Y0);
            }
            m2_batch<N, PRIME, B, Q, M3 + 1>(a, y, xs, lane, hs, p, hb, X0, Y0);
        } else {
            m2_batch<N, PRIME, B, Q + 1, 0>(a, y, xs, lane, hs, p, hb, X0, Y0);
        }
    }
}

// a REST pass (PRIME: REST' of the partner row) into the TMEM row at ta,
// 4 outputs per TMEM access
template <int N, bool PRIME, int B = 0>
__device__ __forceinline__ void m2_pass(uint32_t ta, const double2 (&y)[N], const double2* __restrict__ xs, int lane,
                                        const double2* __restrict__ hs, int& p, double2& hb, double2 X0, double2 Y0) {
    if constexpr (B < N / 4) {
        double2 a[4];
        tm_ld4c(ta + 16 * B, a);
        m2_batch<N, PRIME, B>(a, y, xs, lane, hs, p, hb, X0, Y0);
        tm_st4c(ta + 16 * B, a);
        m2_pass<N, PRIME, B + 1>(ta, y, xs, lane, hs, p, hb, X0, Y0);
    }
}

template <int N>
__global__ void __launch_bounds__(kLanes* kConvWarps, 1)
k_conv_mirror2(const double2* __restrict__ A, double2* __restrict__ B, const double* __restrict__ H,
               const int4* __restrict__ ent, const int* __restrict__ items, const int* __restrict__ order, int ngroups,
               int lpt_from) {
    using PL = Mirror2Layout<N>;
    constexpr int T = N, N3 = N * N * N, COLS = m2_tmem_cols(N);
    extern __shared__ __align__(16) char smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t* tbase_s = reinterpret_cast<uint32_t*>(smem + kConvWarps * PL::WARP_BYTES);
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tbase_s)),
                     "r"(COLS) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tbase_s + ((uint32_t)(32 * (wid & 3)) << 16);
    const uint32_t t_r = tmem, t_rm = tmem + 4 * N;
    const int2 unit = mirror_unit(order, lpt_from);
    const int* it = items + kItemInts * unit.x;
    const int g = unit.y * kConvWarps + wid;
    if (g < ngroups) {
        const int r = __ldg(it), rm = __ldg(it + 1);
        const int e_begin = __ldg(it + 2), e_endI = __ldg(it + 3), e_rm = __ldg(it + 4), e_end = __ldg(it + 5);
        char* wsm = smem + wid * PL::WARP_BYTES;
        unsigned long long* bar = reinterpret_cast<unsigned long long*>(wsm + 3 * PL::X_BYTES + 2 * PL::H_BYTES);
        const double2* ys = reinterpret_cast<const double2*>(wsm + 2 * PL::X_BYTES);
        const double2* Abase = A + (size_t)g * N3 * kLanes;
        double2* Bm = B + ((size_t)g * N3 + (size_t)(rm < 0 ? 0 : rm) * N) * kLanes + lane;
        auto issue = [&](int slot, int4 en) {  // the whole warp (converged)
            const unsigned hb = 8u * (en.w == BT_A ? m2_slab(N, BT_A) : m2_slab(N, BT_FULL));
            if constexpr (BOLTZ_TMA_ELECT) {
                bulk_g2s3_elect(bar + slot, wsm + slot * PL::X_BYTES, Abase + (size_t)en.x * kLanes, PL::X_BYTES,
                                wsm + 2 * PL::X_BYTES, Abase + (size_t)en.y * kLanes, PL::X_BYTES,
                                wsm + 3 * PL::X_BYTES + slot * PL::H_BYTES, H + (size_t)(unsigned)en.z, hb);
            } else if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(bar + slot, 2 * PL::X_BYTES + hb);
                bulk_g2s(wsm + slot * PL::X_BYTES, Abase + (size_t)en.x * kLanes, PL::X_BYTES, bar + slot);
                bulk_g2s(wsm + 2 * PL::X_BYTES, Abase + (size_t)en.y * kLanes, PL::X_BYTES, bar + slot);
                bulk_g2s(wsm + 3 * PL::X_BYTES + slot * PL::H_BYTES, H + (size_t)(unsigned)en.z, hb, bar + slot);
            }
        };
        {   // both TMEM rows start at 0
            const double2 z[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0),
                                  make_double2(0.0, 0.0)};
#pragma unroll
            for (int b = 0; b < N / 4; ++b) {
                tm_st4c(t_r + 16 * b, z);
                tm_st4c(t_rm + 16 * b, z);
            }
            tm_wait_st();
        }
        uint32_t t_cur = t_r;
        double2 acc[T];
#pragma unroll
        for (int i = 0; i < T; ++i) acc[i] = make_double2(0.0, 0.0);
        auto add_tmem = [&](uint32_t ta) {
            tm_wait_st();
#pragma unroll
            for (int b = 0; b < N / 4; ++b) {
                double2 v[4];
                tm_ld4c(ta + 16 * b, v);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    acc[4 * b + q].x += v[q].x;
                    acc[4 * b + q].y += v[q].y;
                }
            }
        };
        auto boundary = [&](int e) {
            if (rm < 0) return;
            if (e == e_endI) {  // I entries done: the conjugate of A(r), k3-reversed, seeds row r'
                Bm[0] = make_double2(0.0, 0.0);
#pragma unroll
                for (int k = 1; k < N; ++k) Bm[(size_t)k * kLanes] = make_double2(acc[N - k].x, -acc[N - k].y);
            }
            if (e == e_rm) {  // row r complete: write it, continue with row r'
                add_tmem(t_r);
                write_row<N, T>(B, g, r, 0, lane, acc);
#pragma unroll
                for (int k = 0; k < N; ++k) acc[k] = Bm[(size_t)k * kLanes];
                t_cur = t_rm;
            }
        };
        if (e_begin < e_end) {
            if (lane == 0) {
                mbar_init(bar, 1);
                mbar_init(bar + 1, 1);
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            }
            __syncwarp();
            EntSrc src(ent, e_begin, e_end, lane);
            int4 en = src.first(e_begin);
            issue(0, en);
            mbar_wait(bar, 0);
            double2 y[T];
#pragma unroll
            for (int j = 0; j < T; ++j) y[j] = ys[j * kLanes + lane];
            for (int e = e_begin; e < e_end; ++e) {
                const int i = e - e_begin, cur = i & 1;
                const bool more = e + 1 < e_end;
                const int4 nx = src.next(e, more, en);
                boundary(e);
                __syncwarp();  // every lane read y (registers) and is done with slot cur^1
                if (more) issue(cur ^ 1, nx);
                const double2* xs = reinterpret_cast<const double2*>(wsm + cur * PL::X_BYTES);
                const double2* hs = reinterpret_cast<const double2*>(wsm + 3 * PL::X_BYTES + cur * PL::H_BYTES);
                auto xat = [&](int m3) { return xs[m3 * kLanes + lane]; };
                auto none = [](int, int) {};
                {
                    int p = 0;
                    double2 hb = make_double2(0.0, 0.0);
                    band_tile<N, T, 1, 0, 0, BT_A>(acc, y, xat, hs, p, hb, none);
                }
                const double2 zero = make_double2(0.0, 0.0);
                tm_wait_st();  // the previous entry's TMEM stores
                int pr = 0;
                double2 hbr = zero;
                if (en.w == BT_A) {  // interior input rows: REST of r and REST' of r'
                    const int m1 = en.x / (N * N), m2 = (en.x / N) % N, s1 = en.y / (N * N), s2 = (en.y / N) % N;
                    const double2 X0 = ldg2(Abase + (size_t)(((N - m1) * N + (N - m2)) * N) * kLanes + lane);
                    const double2 Y0 = ldg2(Abase + (size_t)(((N - s1) * N + (N - s2)) * N) * kLanes + lane);
                    m2_pass<N, false>(t_r, y, xs, lane, hs + m2_a(N) / 2, pr, hbr, zero, zero);
                    int pp = 0;
                    double2 hbp = zero;
                    m2_pass<N, true>(t_rm, y, xs, lane, hs + (m2_a(N) + m2_r(N)) / 2, pp, hbp, X0, Y0);
                } else {  // FULL: the REST band into the registers too
                    band_tile<N, T, 1, 0, 0, BT_REST>(acc, y, xat, hs + m2_a(N) / 2, pr, hbr, none);
                }
                if (more) {
                    mbar_wait(bar + (cur ^ 1), (unsigned)(((i + 1) >> 1) & 1));
#pragma unroll
                    for (int j = 0; j < T; ++j) y[j] = ys[j * kLanes + lane];
                }
                en = nx;
            }
        }
        boundary(e_end);  // boundaries that coincide with the end of the list
        add_tmem(t_cur);
        write_row<N, T>(B, g, rm >= 0 ? rm : r, 0, lane, acc);
    }
    tm_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (wid == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tbase_s), "r"(COLS) : "memory");
}

// ---------------------------------------------------------------------------
// k_conv_kcsm (N = 24, 32: the k-chunked kcs kernels, TMA staging): the
// Hermitian mirror schedule in two phases, so that each kernel still unrolls
// one k-chunk's code.  The k3 reversal maps chunk KC of row r onto chunk
// NK-1-KC of r' = N - r, which a kernel of chunk KC cannot sum, so:
//   phase 0 (one launch per KC, rows = pair leaders r < r'): sums A(r) over the
//     interior input rows and writes it, raw, to chunk KC of row r of B, and
//     its conjugate, k3-reversed, to row r' (B[r'][N - k3] = conj A[r][k3]);
//   phase 1 (one launch per KC, rows = pair rows): adds the REST entries
//     (the rest of the interior input rows' terms) to the seed in B, raw;
//   phase 2 (one launch per KC, rows = every output row): starts from B (pair
//     rows) or 0, adds the FULL entries and writes the chunk with s_k.
// Launch order: phase 0, 1, 2, each over KC = 0..NK-1; every launch unrolls
// one band type of one chunk.  Without kcsm_split, phase 3 replaces 1 and 2
// (REST and FULL entries of every row, typed per entry, one launch).  Slab of an entry
// of type ty for chunk KC at H + en.z + KC * kcsm_slab(N, ty): one even-padded
// piece per tile, in band_tile order.
// list = [CSR offsets (nrows + 1) | output row (nrows) | aux (nrows) |
//         longest-first order (nrows)], aux = partner r' (phase 0) or
//         1 if the row is seeded from B (phases 1, 2).
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int even_up(int c) { return (c + 1) & ~1; }
__host__ __device__ constexpr int tile_terms_t(int n, int t, int kc, int ti, int ty) {
    const int nk = n / t, sc = band_tile_sc(nk, kc, ti);
    int c = 0;
    for (int m3 = 0; m3 < n; ++m3)
        for (int kk = 0; kk < t; ++kk) c += band_term_t(n, t, kc, sc, m3, kk, ty) ? 1 : 0;
    return c;
}
// offset (doubles) of tile ti's piece within a chunk slab of type ty
__host__ __device__ constexpr int kcsm_piece_off(int n, int t, int kc, int ti, int ty) {
    int o = 0;
    for (int u = 0; u < ti; ++u) o += even_up(tile_terms_t(n, t, kc, u, ty));
    return o;
}
__host__ __device__ constexpr int kcsm_slab_kc(int n, int t, int kc, int ty) { return kcsm_piece_off(n, t, kc, n / t, ty); }
// per-chunk stride of an entry's slab (max over chunks)
__host__ __device__ constexpr int kcsm_slab(int n, int ty) {
    const int t = conv_tile(n);
    int mx = 0;
    for (int kc = 0; kc < n / t; ++kc) mx = kcsm_slab_kc(n, t, kc, ty) > mx ? kcsm_slab_kc(n, t, kc, ty) : mx;
    return mx;
}

// ---------------------------------------------------------------------------
// The REST fold (N = 32, BOLTZ_KCSF): kernel phase 4 = phase 0 of k_conv_kcsm
// with the pair rows' REST terms folded in; it replaces k_conv_kcsr.  An entry
// of a pair leader r (interior input row m, y row s staged) also sums, between
// its two tiles, the chunk's REST terms of r and the REST' terms of the
// partner r' = N - r -- r''s own non-mirrored terms, from r's rows: x'[m3'] =
// conj x[N - m3'], x'[0] = fhat(N - m1, N - m2, 0), likewise y' (as
// k_conv_mirror2's REST') -- k3-major, 4 outputs per TMEM access, into two TMEM
// rows of 16 complex values per warp.  The REST terms then reuse the staged y
// row and the x row the A band just read, instead of restaging both per REST
// entry (k_conv_kcsr: ~33 KB of L2 per 109 terms, FP64 pipe 52%).
// Epilogue: chunk KC of row r = A + T_r; row r' takes conj(A) at N - k3 and
// T_r' at k3' (the KC = 0 launch writes the row, KC = 1 adds to it).
// Slab of an entry, per chunk: [A pieces | REST(r) | REST'(r'), flagged].
// Measured on B200 and left off (BOLTZ_KCSF=1 opts in; bitwise-equal checksum,
// oracle parity green): cfg5-shaped collide at 2048 cells 145.1 -> 164.2 ms.
// ncu: phase 4 takes 59.7 / 53.7 ms (chunk 0 / 1) against 27.6 + 32.9 for
// phase 0 plus 30.1 for k_conv_kcsr -- the REST passes run at ~3x the A band's
// cost per term: each term's x comes from L1/L2 right before its use (long
// scoreboard 16%), every 4-output batch waits on its tcgen05.ld, and the extra
// code spills (160 / 400 B) and misses the I-cache (no_instructions 7%).
// ---------------------------------------------------------------------------
#ifndef BOLTZ_KCSF
#define BOLTZ_KCSF 0
#endif
// REST terms of chunk kc (k3 in [kc T, kc T + T))
__host__ __device__ constexpr int kcsf_rest_kc(int n, int kc) {
    const int t = conv_tile(n);
    int c = 0;
    for (int k3 = kc * t; k3 < kc * t + t; ++k3)
        for (int m3 = 0; m3 < n; ++m3) c += rest_term(n, k3, m3) ? 1 : 0;
    return c;
}
__host__ __device__ constexpr int kcsf_a_kc(int n, int kc) { return kcsm_slab_kc(n, conv_tile(n), kc, BT_A); }
__host__ __device__ constexpr int kcsf_slab_kc(int n, int kc) {
    return kcsf_a_kc(n, kc) + 2 * even_up(kcsf_rest_kc(n, kc));
}
// per-chunk stride of a phase-4 entry's slab
__host__ __device__ constexpr int kcsf_slab(int n) {
    int mx = 0;
    for (int kc = 0; kc < n / conv_tile(n); ++kc) mx = kcsf_slab_kc(n, kc) > mx ? kcsf_slab_kc(n, kc) : mx;
    return mx;
}
// the phase whose band code a kernel phase runs (4: phase 0's A band)
__host__ __device__ constexpr int kcsm_ph(int phase) { return phase == 4 ? 0 : phase; }

// per-warp shared memory of phase PHASE (its H slots sized for its band type;
// phase 3 holds REST or FULL slabs, phase 4 the folded slabs)
template <int N, int PHASE = 3>
struct KcsmLayout {
    static constexpr int T = conv_tile(N);
    static constexpr int NK = N / T;
    static constexpr int Y_BYTES = N * kLanes * 16;
    static constexpr int H_BYTES =
        (PHASE == 4 ? kcsf_slab(N) : kcsm_slab(N, PHASE == 0 ? (int)BT_A : PHASE == 1 ? (int)BT_REST : (int)BT_FULL)) * 8;
    static constexpr int WARP_BYTES = Y_BYTES + 2 * H_BYTES + 16;  // + 2 mbarriers
    static constexpr int TMEM_BYTES = PHASE == 4 ? 16 : 0;         // the CTA's TMEM base address
};
// cell groups (warps) per CTA of k_conv_kcsm: 8 at N=24 (cfg4 RK2 step 31.3 ->
// 30.4 ms), the global kConvWarps elsewhere (8 measured +7% at N=32)
#ifndef BOLTZ_KCSM_WARPS24
#define BOLTZ_KCSM_WARPS24 8
#endif
__host__ __device__ constexpr int kcsm_warps(int n) { return n == 24 ? BOLTZ_KCSM_WARPS24 : kConvWarps; }
#ifndef BOLTZ_KCSM_REST_MINB
#define BOLTZ_KCSM_REST_MINB 1  // CTAs per SM the REST phase is compiled for (registers)
#endif

// the band type phase PHASE runs: 0 the pair leaders' A terms, 1 REST, 2 FULL,
// 3 REST or FULL per entry (phases 1 and 2 in one launch)
__host__ __device__ constexpr int kcsm_type(int phase) {
    return phase == 0 || phase == 4 ? BT_A : phase == 1 ? BT_REST : BT_FULL;
}
// phases 1 and 2 as separate launches (one band type unrolled per kernel) for
// two k-chunks; one launch at N=24 (measured: N=32 339.8 -> 330.7 ms per RK2
// step split, N=24 31.3 -> 32.8 ms)
#ifndef BOLTZ_KCSM_SPLIT
#define BOLTZ_KCSM_SPLIT -1  // -1: split for two k-chunks; 0 / 1 force (tuning)
#endif
__host__ __device__ constexpr bool kcsm_split(int n) {
    return BOLTZ_KCSM_SPLIT >= 0 ? BOLTZ_KCSM_SPLIT == 1 : n / conv_tile(n) > 1;
}
// N = 32: the REST fold (kernel phase 4) instead of k_conv_kcsr
__host__ __device__ constexpr bool kcsf_n(int n) { return BOLTZ_KCSF && n == 32 && kcsm_split(n); }

// one tile of a k_conv_kcsm entry on the y window in registers (x per
// diagonal from L2)
// Gauss term form per k_conv_kcsm kernel, by measurement on B200 (ncu launch
// list, 2048 cells): <32,0,0> 29.3 -> 27.4 ms, <32,0,2> 27.7 -> 24.9 ms,
// <32,0,1> 25.2 -> 25.5; the KC = 1 kernels and N = 24 spill registers with it
// (84-896 B of stack) and run slower, so they keep the 6-instruction term.
#ifndef BOLTZ_KCSM_GAUSS
#define BOLTZ_KCSM_GAUSS 1
#endif
// chunk-1 kernels (kc = 1, N = 32): kk passes of the band (band_tile KS) and the
// Gauss form there (dev knobs, off): the passes do not relieve the registers --
// ptxas: KS = 2 255 registers + 72 B stack; KS = 2 + Gauss 255 + 536 B; Gauss
// alone 255 + 64 / 112 B (the 6-instruction term: 244 / 242, no stack)
#ifndef BOLTZ_KCSM_KS1
#define BOLTZ_KCSM_KS1 1
#endif
#ifndef BOLTZ_KCSM_GAUSS1
#define BOLTZ_KCSM_GAUSS1 0
#endif
__host__ __device__ constexpr int kcsm_ks(int n, int kc, int ty) {
    return (n == 32 && kc == 1 && (ty == BT_A || ty == BT_FULL)) ? BOLTZ_KCSM_KS1 : 1;
}
__host__ __device__ constexpr bool kcsm_gauss(int n, int kc, int phase) {
    return BOLTZ_TERM_GAUSS || (BOLTZ_KCSM_GAUSS && n == 32 && kc == 0 && (kcsm_ph(phase) == 0 || phase == 2)) ||
           (BOLTZ_KCSM_GAUSS1 && n == 32 && kc == 1 && (kcsm_ph(phase) == 0 || phase == 2));
}
template <int N, int KC, int PHASE>
using KcsmY = std::conditional_t<kcsm_gauss(N, KC, PHASE), YG, double2>;
template <typename YT>
__device__ __forceinline__ YT to_yt(double2 v) {
    if constexpr (std::is_same<YT, YG>::value) return to_yg(v);
    else return v;
}

template <int N, int KC, int TI, int PHASE, typename YT>
__device__ __forceinline__ void kcsm_tile(double2 (&acc)[conv_tile(N)], const YT (&y)[conv_tile(N)],
                                          const double2* X, const double2* hs, int ty) {
    constexpr int T = conv_tile(N), NK = N / T;
    auto xat = [&](int m3) { return ldg2(X + (size_t)m3 * kLanes); };
    auto none = [](int, int) {};
    double2 hb = make_double2(0.0, 0.0);
    int p = 0;
    if constexpr (PHASE < 3 || PHASE == 4) {
        constexpr int TY = kcsm_type(PHASE);
        band_tile<N, T, NK, KC, TI, TY, kcsm_ks(N, KC, TY)>(acc, y, xat, hs + kcsm_piece_off(N, T, KC, TI, TY) / 2, p,
                                                           hb, none);
    } else if (ty == BT_FULL) {
        band_tile<N, T, NK, KC, TI, BT_FULL>(acc, y, xat, hs + kcsm_piece_off(N, T, KC, TI, BT_FULL) / 2, p, hb, none);
    } else {
        band_tile<N, T, NK, KC, TI, BT_REST>(acc, y, xat, hs + kcsm_piece_off(N, T, KC, TI, BT_REST) / 2, p, hb, none);
    }
}

// one REST (PRIME: REST' of the partner row) term of the fold: x from L2 (the
// row the A band just read), y from the staged row
template <int N, bool PRIME, int K3, int M3>
__device__ __forceinline__ void kf_term(double2& a, double h, const double2* __restrict__ X,
                                        const double2* __restrict__ ys, int lane, double2 X0, double2 Y0) {
    constexpr int S3 = K3 - M3 + N / 2;
    auto xg = [&](int m) { return ldg2(X + (size_t)m * kLanes); };
    auto yg = [&](int s) { return ys[s * kLanes + lane]; };
    if constexpr (!PRIME) {
        const double2 xm = xg(M3), yv = yg(S3);
        const double tr = fma(xm.x, yv.x, -xm.y * yv.y);
        const double ti = fma(xm.x, yv.y, xm.y * yv.x);
        a.x = fma(h, tr, a.x);
        a.y = fma(h, ti, a.y);
    } else if constexpr (M3 == 0) {  // X0 * conj(y[N - s3])  (s3 >= 1 here)
        const double2 yv = yg((N - S3) % N);
        const double tr = fma(X0.x, yv.x, X0.y * yv.y);
        const double ti = fma(X0.y, yv.x, -X0.x * yv.y);
        a.x = fma(h, tr, a.x);
        a.y = fma(h, ti, a.y);
    } else if constexpr (S3 == 0) {  // conj(x[N - m3]) * Y0
        const double2 xm = xg(N - M3);
        const double tr = fma(xm.x, Y0.x, xm.y * Y0.y);
        const double ti = fma(xm.x, Y0.y, -xm.y * Y0.x);
        a.x = fma(h, tr, a.x);
        a.y = fma(h, ti, a.y);
    } else {  // conj(x[N - m3] * y[N - s3])
        const double2 xm = xg(N - M3), yv = yg(N - S3);
        const double tr = fma(xm.x, yv.x, -xm.y * yv.y);
        const double ti = fma(xm.x, yv.y, xm.y * yv.x);
        a.x = fma(h, tr, a.x);
        a.y = fma(-h, ti, a.y);
    }
}
// the REST terms of outputs k3 = KC T + 4B .. +3 into a[4] (slab order: B, Q, m3)
template <int N, int KC, bool PRIME, int B, int Q = 0, int M3 = 0>
__device__ __forceinline__ void kf_batch(double2 (&a)[4], const double2* __restrict__ X,
                                         const double2* __restrict__ ys, int lane, const double2* __restrict__ hs,
                                         int& p, double2& hb, double2 X0, double2 Y0) {
    constexpr int K3 = KC * conv_tile(N) + 4 * B + Q;
    if constexpr (Q < 4) {
        if constexpr (M3 < N) {
            if constexpr (rest_term(N, K3, M3)) {
                double h;
                if ((p & 1) == 0) { hb = hs[p >> 1]; h = hb.x; }
                else h = hb.y;
                ++p;
                kf_term<N, PRIME, K3, M3>(a[Q], h, X, ys, lane, X0, Y0);
            }
            kf_batch<N, KC, PRIME, B, Q, M3 + 1>(a, X, ys, lane, hs, p, hb, X0, Y0);
        } else {
            kf_batch<N, KC, PRIME, B, Q + 1, 0>(a, X, ys, lane, hs, p, hb, X0, Y0);
        }
    }
}
// a REST pass of chunk KC into the TMEM row at ta, 4 outputs per TMEM access
template <int N, int KC, bool PRIME, int B = 0>
__device__ __forceinline__ void kf_pass(uint32_t ta, const double2* __restrict__ X, const double2* __restrict__ ys,
                                        int lane, const double2* __restrict__ hs, int& p, double2& hb, double2 X0,
                                        double2 Y0) {
    if constexpr (B < conv_tile(N) / 4) {
        double2 a[4];
        tm_ld4c(ta + 16 * B, a);
        kf_batch<N, KC, PRIME, B>(a, X, ys, lane, hs, p, hb, X0, Y0);
        tm_st4c(ta + 16 * B, a);
        kf_pass<N, KC, PRIME, B + 1>(ta, X, ys, lane, hs, p, hb, X0, Y0);
    }
}

// WW: cell groups (warps) per CTA -- kcsm_warps(N), or kConvWarps at N = 24 for
// batches of at most kConvWarps groups, where 8-warp CTAs would run half empty
template <int N, int KC, int PHASE, int WW = kcsm_warps(N)>
__global__ void __launch_bounds__(kLanes* WW, PHASE == 1 ? BOLTZ_KCSM_REST_MINB : BOLTZ_K0_MINB)
k_conv_kcsm(const double2* __restrict__ A, double2* __restrict__ B, const double* __restrict__ H,
            const int4* __restrict__ ent, const int* __restrict__ list, int nrows, int ngroups, int lpt_from, int head_lpt) {
    using LY = KcsmLayout<N, PHASE>;
    constexpr int T = LY::T, NK = LY::NK, N3 = N * N * N, W = WW;
    constexpr bool FOLD = PHASE == 4;
    static_assert(!FOLD || (T % 4 == 0 && W <= 4), "the fold: 4-output TMEM batches, one TMEM lane quarter per warp");
    constexpr int PH = kcsm_ph(PHASE);
    // this chunk's part of an entry's slab (phase 3: REST or FULL per entry; phase 4: the folded slab)
    constexpr int TY = kcsm_type(PHASE == 3 ? 2 : PHASE);
    constexpr size_t OFF = (size_t)KC * (FOLD ? kcsf_slab(N) : kcsm_slab(N, TY)), OFF_R = (size_t)KC * kcsm_slab(N, BT_REST);
    constexpr unsigned BYTES = 8u * (FOLD ? kcsf_slab_kc(N, KC) : kcsm_slab_kc(N, T, KC, TY)),
                       BYTES_R = 8u * kcsm_slab_kc(N, T, KC, BT_REST);
    extern __shared__ __align__(16) char smem[];
    const int2 unit = lpt_unit(list + 3 * nrows + 1, lpt_from, head_lpt);
    const int wi = unit.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int g = unit.y * W + wid;
    // phase 4: two TMEM rows (REST of r, REST' of r') of T complex values per warp
    [[maybe_unused]] uint32_t* tbase_s = reinterpret_cast<uint32_t*>(smem + W * LY::WARP_BYTES);
    [[maybe_unused]] constexpr int COLS = FOLD ? (8 * T <= 32 ? 32 : 8 * T <= 64 ? 64 : 8 * T <= 128 ? 128 : 256) : 0;
    if constexpr (FOLD) {
        if (wid == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tbase_s)),
                         "r"(COLS) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    if (g < ngroups) {
    const int row = __ldg(list + nrows + 1 + wi), aux = __ldg(list + 2 * nrows + 1 + wi);
    const int e0 = __ldg(list + wi), e1 = __ldg(list + wi + 1);
    char* wsm = smem + wid * LY::WARP_BYTES;
    double2* ys = reinterpret_cast<double2*>(wsm);
    char* hbase = wsm + LY::Y_BYTES;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(wsm + LY::Y_BYTES + 2 * LY::H_BYTES);
    const double2* Abase = A + (size_t)g * N3 * kLanes;
    const double2* Ag = Abase + lane;
    double2* Brow = B + ((size_t)g * N3 + (size_t)row * N + KC * T) * kLanes + lane;
    [[maybe_unused]] uint32_t t_r = 0, t_rm = 0;
    if constexpr (FOLD) {
        t_r = *tbase_s + ((uint32_t)(32 * (wid & 3)) << 16);
        t_rm = t_r + 4 * T;
        const double2 z[4] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0), make_double2(0.0, 0.0),
                              make_double2(0.0, 0.0)};
#pragma unroll
        for (int b = 0; b < T / 4; ++b) {
            tm_st4c(t_r + 16 * b, z);
            tm_st4c(t_rm + 16 * b, z);
        }
    }
    double2 acc[T];
    if (PH >= 1 && aux) {
#pragma unroll
        for (int kk = 0; kk < T; ++kk) acc[kk] = Brow[(size_t)kk * kLanes];
    } else {
#pragma unroll
        for (int kk = 0; kk < T; ++kk) acc[kk] = make_double2(0.0, 0.0);
    }
    auto tma_h = [&](int slot, int4 en) {  // the whole warp (converged)
        const bool rest = PHASE == 3 && en.w == BT_REST;
        const unsigned bytes = rest ? BYTES_R : BYTES;
        if constexpr (BOLTZ_TMA_ELECT) {
            bulk_g2s1_elect(bar + slot, hbase + slot * LY::H_BYTES, H + (size_t)(unsigned)en.z + (rest ? OFF_R : OFF),
                            bytes);
        } else if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar + slot, bytes);
            bulk_g2s(hbase + slot * LY::H_BYTES, H + (size_t)(unsigned)en.z + (rest ? OFF_R : OFF), bytes, bar + slot);
        }
    };
    auto tma_y = [&](int slot, int4 en) {  // the whole warp (converged)
        if constexpr (BOLTZ_TMA_ELECT) {
            bulk_g2s1_elect(bar + slot, ys, Abase + (size_t)en.y * kLanes, LY::Y_BYTES);
        } else if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar + slot, LY::Y_BYTES);
            bulk_g2s(ys, Abase + (size_t)en.y * kLanes, LY::Y_BYTES, bar + slot);
        }
    };
    // phase 4: the chunk's REST of r and REST' of r' from the staged rows
    auto rest_fold = [&](int4 en, const double2* X, const double2* hs) {
        if constexpr (FOLD) {
            const int m1 = en.x / (N * N), m2 = (en.x / N) % N, s1 = en.y / (N * N), s2 = (en.y / N) % N;
            const double2 X0 = ldg2(Abase + (size_t)(((N - m1) * N + (N - m2)) * N) * kLanes + lane);
            const double2 Y0 = ldg2(Abase + (size_t)(((N - s1) * N + (N - s2)) * N) * kLanes + lane);
            const double2 zero = make_double2(0.0, 0.0);
            tm_wait_st();  // the previous entry's TMEM stores
            int p = 0;
            double2 hb = zero;
            kf_pass<N, KC, false>(t_r, X, ys, lane, hs + kcsf_a_kc(N, KC) / 2, p, hb, zero, zero);
            int pp = 0;
            double2 hbp = zero;
            kf_pass<N, KC, true>(t_rm, X, ys, lane, hs + (kcsf_a_kc(N, KC) + even_up(kcsf_rest_kc(N, KC))) / 2, pp,
                                 hbp, X0, Y0);
        }
    };
    if (e0 < e1) {
        if (lane == 0) {
            mbar_init(bar, 2);
            mbar_init(bar + 1, 2);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        std::conditional_t<BOLTZ_KCSM_ENTWIN && N == 32, EntWin, EntAhead> src(ent, e0, e1, lane);
        int4 en = src.first(e0);
        tma_y(0, en);
        tma_h(0, en);
        mbar_wait(bar, 0);
        for (int e = e0; e < e1; ++e) {
            const int i = e - e0, cur = i & 1;
            const bool more = e + 1 < e1;
            const int4 nx = src.next(e, more, en);
            __syncwarp();  // every lane finished reading H[cur^1]
            if (more) tma_h(cur ^ 1, nx);
            const double2* X = Ag + (size_t)en.x * kLanes;
            const double2* hs = reinterpret_cast<const double2*>(hbase + cur * LY::H_BYTES);
            KcsmY<N, KC, PHASE> y[T];
#pragma unroll
            for (int j = 0; j < T; ++j) y[j] = to_yt<KcsmY<N, KC, PHASE>>(ys[(band_tile_sc(NK, KC, 0) * T + j) * kLanes + lane]);
            if constexpr (NK == 1) {
                rest_fold(en, X, hs);  // (phase 4 needs the y row: before the refill)
                __syncwarp();  // every lane holds its y window: the buffer may be refilled
                if (more) tma_y(cur ^ 1, nx);
                kcsm_tile<N, KC, 0, PHASE>(acc, y, X, hs, en.w);
            } else {
                kcsm_tile<N, KC, 0, PHASE>(acc, y, X, hs, en.w);
                rest_fold(en, X, hs);  // between the tiles: the y row is still staged
#pragma unroll
                for (int j = 0; j < T; ++j) y[j] = to_yt<KcsmY<N, KC, PHASE>>(ys[(band_tile_sc(NK, KC, 1) * T + j) * kLanes + lane]);
                __syncwarp();
                if (more) tma_y(cur ^ 1, nx);
                kcsm_tile<N, KC, (NK > 1 ? 1 : 0), PHASE>(acc, y, X, hs, en.w);
            }
            if (more) mbar_wait(bar + (cur ^ 1), (unsigned)(((i + 1) >> 1) & 1));
            en = nx;
        }
    }
    if constexpr (PHASE == 0) {
        // raw A(r) of chunk KC; conj seeds k3' = N - k3 of the partner (k3' = 0: none)
#pragma unroll
        for (int kk = 0; kk < T; ++kk) Brow[(size_t)kk * kLanes] = acc[kk];
        double2* Bm = B + ((size_t)g * N3 + (size_t)aux * N) * kLanes + lane;
#pragma unroll
        for (int kk = 0; kk < T; ++kk) {
            const int k3 = KC * T + kk;
            if (k3 != 0) Bm[(size_t)(N - k3) * kLanes] = make_double2(acc[kk].x, -acc[kk].y);
        }
        if (KC == NK - 1) Bm[0] = make_double2(0.0, 0.0);
    } else if constexpr (FOLD) {
        // row r, chunk KC: A + REST(r), raw (phase 2 continues it)
        tm_wait_st();
#pragma unroll
        for (int b = 0; b < T / 4; ++b) {
            double2 v[4];
            tm_ld4c(t_r + 16 * b, v);
#pragma unroll
            for (int q = 0; q < 4; ++q)
                Brow[(size_t)(4 * b + q) * kLanes] = make_double2(acc[4 * b + q].x + v[q].x, acc[4 * b + q].y + v[q].y);
        }
        // row r': conj(A) k3-reversed (k3' = N - k3, none for k3 = 0) and REST'(r') at k3' = KC T + kk; the
        // first chunk's launch writes the row (k3' = N/2 .. : zero where nothing lands yet), later ones add
        double2* Bm = B + ((size_t)g * N3 + (size_t)aux * N) * kLanes + lane;
        double2 tv[T];
#pragma unroll
        for (int b = 0; b < T / 4; ++b) {
            double2 v[4];
            tm_ld4c(t_rm + 16 * b, v);
#pragma unroll
            for (int q = 0; q < 4; ++q) tv[4 * b + q] = v[q];
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
            double2 v = KC == 0 ? make_double2(0.0, 0.0) : Bm[(size_t)k * kLanes];
            const int kk = N - k - KC * T;  // conj A[k3 = N - k] of this chunk
            if (k != 0 && kk >= 0 && kk < T) {
                v.x += acc[kk].x;
                v.y -= acc[kk].y;
            }
            if (k >= KC * T && k < KC * T + T) {  // REST'(r') at k3' = k
                v.x += tv[k - KC * T].x;
                v.y += tv[k - KC * T].y;
            }
            Bm[(size_t)k * kLanes] = v;
        }
    } else if constexpr (PHASE == 1) {  // seed + REST, raw: phase 2 continues the row
#pragma unroll
        for (int kk = 0; kk < T; ++kk) Brow[(size_t)kk * kLanes] = acc[kk];
    } else {
        write_row<N, T>(B, g, row, KC, lane, acc);
    }
    }  // g < ngroups
    if constexpr (FOLD) {
        tm_wait_st();
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (wid == 0)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tbase_s), "r"(COLS) : "memory");
    }
}

// ---------------------------------------------------------------------------
// k_conv_kcsr (N = 32, replaces phase 1 of k_conv_kcsm): the REST entries of
// the pair rows for BOTH k-chunks in one launch.  A REST entry holds few terms
// (the non-interior ones and the k3 = 0 column: 109 at N = 32, against ~700
// A terms) but needs the whole x and y rows, so phase 1 ran one L2-bound pass
// per k-chunk.  Here an entry's rows are staged once for the full output row:
// 32 accumulators in registers, x per diagonal from L2, the H slab by TMA
// (double-buffered) and the y row by TMA into a single buffer, read in three
// parts so that the buffer is refilled early:
//   part 0: the edge diagonals m3 in {0, 1, N-1} (y per term from smem)
//   part 1: the k3 = 0 column of the interior diagonals (y per term from smem)
//   -- y[0], y[1], y[N-1] to registers; the next entry's y row is issued --
//   part 2: the interior diagonals' remaining terms, whose s3 is 0, 1 or N-1
// The table builder lays the slab out in exactly this order (kcsr_part).  The
// row is seeded from B (phase 0's raw A or its mirror) and written back raw;
// phase 2 finishes it.  Per-cell order is fixed: bitwise batch-independent.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr bool kcsr_term(int n, int k3, int m3) {
    const int s3 = k3 - m3 + n / 2;
    return s3 >= 0 && s3 < n && type_term(n, BT_REST, k3, m3);
}
// y buffers per warp: 1 -- the three parts above; 2 -- double-buffered y row
// and one diagonal-major pass (every term in part 0).  B200, cfg5-shaped RK2
// step (2048 cells), K2 ms: phase 1 per k-chunk 318.0 | kcsr 1 buffer, 4 warps
// 305.8 | 2 buffers, 2 warps per CTA 299.9 | 3 warps 301.9 | 4 warps 322.5
// 4 -- k_conv_kcsrq: one y row refilled by quarters (below; measured no gain)
#ifndef BOLTZ_KCSR_YBUF
#define BOLTZ_KCSR_YBUF 2
#endif
// with 2 y buffers: part 2's y[0], y[1], y[N-1] from registers (44 of the 109
// terms) instead of shared memory -- the kernel is shared-memory-bandwidth-bound
#ifndef BOLTZ_KCSR_YREG
#define BOLTZ_KCSR_YREG 0  // measured: 310.3 against 299.9 ms per RK2 step (255 registers, 32 B spilled)
#endif
// is REST term (k3, m3) in part `part` (0, 1, 2; see above)?
__host__ __device__ constexpr bool kcsr_part(int n, int part, int k3, int m3) {
    if (!kcsr_term(n, k3, m3)) return false;
    if (BOLTZ_KCSR_YBUF >= 2 && !BOLTZ_KCSR_YREG) return part == 0;
    const bool edge = !mirror_interior(n, m3);
    return part == 0 ? edge : part == 1 ? (!edge && k3 == 0) : (!edge && k3 != 0);
}
__host__ __device__ constexpr int kcsr_slab(int n) {
    int c = 0;
    for (int m3 = 0; m3 < n; ++m3)
        for (int k3 = 0; k3 < n; ++k3) c += kcsr_term(n, k3, m3) ? 1 : 0;
    return even_up(c);
}
__host__ __device__ constexpr bool kcsr_diag(int n, int part, int m3) {
    bool any = false;
    for (int k3 = 0; k3 < n; ++k3) any = any || kcsr_part(n, part, k3, m3);
    return any;
}
#ifndef BOLTZ_KCSR
#define BOLTZ_KCSR 1  // N = 32: one full-row REST launch instead of phase 1 per k-chunk
#endif
__host__ __device__ constexpr bool kcsr_n(int n) { return BOLTZ_KCSR && !kcsf_n(n) && n == 32 && kcsm_split(n); }
#ifndef BOLTZ_KCSR_WARPS
#define BOLTZ_KCSR_WARPS 2
#endif
constexpr int kKcsrWarps = BOLTZ_KCSR_WARPS;
// term order: see KcsrTab
#ifndef BOLTZ_KCSR_ORDER
#define BOLTZ_KCSR_ORDER 2
#endif
template <int N>
struct KcsrLayout {
    static constexpr int Y_BYTES = N * kLanes * 16;
    static constexpr int H_BYTES = kcsr_slab(N) * 8;
    // ORDER 2: the edge diagonals' x (m3 = 0, 1, N-1) are staged with the y row
    static constexpr int XE_BYTES = (BOLTZ_KCSR_ORDER == 2 && BOLTZ_KCSR_YBUF == 2) ? 3 * kLanes * 16 : 0;
    static constexpr int WARP_BYTES = BOLTZ_KCSR_YBUF * (Y_BYTES + XE_BYTES) + 2 * H_BYTES + 16;  // + 2 mbarriers
};
#ifndef BOLTZ_KCSR_MINB
#define BOLTZ_KCSR_MINB 2
#endif

// the kcsr term list as a compile-time table, in the kernel's visiting order.
// Per term: where x comes from (xsrc 0/1/2: the edge diagonals m3 = 0, 1, N-1
// held in registers for the whole entry; 3: xm, loaded when xload) and where y
// comes from (ysrc 0/1/2: y[0], y[1], y[N-1] in registers; 3: yc, loaded from
// the staged row when yload).
//   BOLTZ_KCSR_ORDER 1: diagonal-major by part (x per diagonal, y per term)
//   BOLTZ_KCSR_ORDER 2: s3-major over the edge diagonals, so that one staged
//     y[s3] feeds every edge term on it and the k3 = 0 term that needs it,
//     whose diagonal's other terms follow (y from registers); then the
//     remaining interior diagonals.  45 -> 32 y loads + 3, against 109.
template <int N>
struct KcsrTab {
    static constexpr int cnt() {
        int c = 0;
        for (int m3 = 0; m3 < N; ++m3)
            for (int k3 = 0; k3 < N; ++k3) c += kcsr_term(N, k3, m3) ? 1 : 0;
        return c;
    }
    static constexpr int COUNT = cnt();
    static constexpr int yreg(int s3) { return s3 == 0 ? 0 : s3 == 1 ? 1 : s3 == N - 1 ? 2 : 3; }
    static constexpr int xreg(int m3) { return m3 == 0 ? 0 : m3 == 1 ? 1 : m3 == N - 1 ? 2 : 3; }
    short k3[COUNT] = {}, m3[COUNT] = {}, part[COUNT] = {};
    signed char xsrc[COUNT] = {}, ysrc[COUNT] = {};
    bool xload[COUNT] = {}, yload[COUNT] = {};
    // k_conv_kcsrq: first / one-past-last term loading the staged y of quarter q (s3 in [qN/4, (q+1)N/4))
    int qbeg[4] = {}, qend[4] = {};
    bool done[N * N] = {};
    int c = 0;
    constexpr void emit(int k, int m, int pt) {
        k3[c] = (short)k;
        m3[c] = (short)m;
        part[c] = (short)pt;
        done[m * N + k] = true;
        ++c;
    }
    constexpr KcsrTab() {
        if (BOLTZ_KCSR_ORDER == 2 && BOLTZ_KCSR_YBUF >= 2) {
            const int edges[3] = {0, 1, N - 1};
            for (int s = 0; s < N; ++s) {
                for (int e = 0; e < 3; ++e) {
                    const int m = edges[e], k = s + m - N / 2;
                    if (k >= 0 && k < N && kcsr_term(N, k, m)) emit(k, m, 2);
                }
                if (yreg(s) != 3) continue;
                for (int m = 2; m <= N - 2; ++m) {  // interior terms on this staged y[s]
                    const int k = s + m - N / 2;
                    if (k < 0 || k >= N || !kcsr_term(N, k, m) || done[m * N + k]) continue;
                    emit(k, m, 2);
                    for (int k2 = 0; k2 < N; ++k2)  // the rest of diagonal m: y from registers
                        if (kcsr_term(N, k2, m) && !done[m * N + k2] && yreg(k2 - m + N / 2) != 3) emit(k2, m, 2);
                }
            }
            for (int m = 0; m < N; ++m)
                for (int k = 0; k < N; ++k)
                    if (kcsr_term(N, k, m) && !done[m * N + k]) emit(k, m, 2);
        } else {
            for (int pt = 0; pt < 3; ++pt)
                for (int m = 0; m < N; ++m)
                    for (int k = 0; k < N; ++k)
                        if (kcsr_part(N, pt, k, m)) emit(k, m, pt);
        }
        const bool regs = BOLTZ_KCSR_ORDER == 2 && BOLTZ_KCSR_YBUF >= 2;
        int xm = -1, yc = -1;
        for (int i = 0; i < COUNT; ++i) {
            const int s = k3[i] - m3[i] + N / 2;
            xsrc[i] = (signed char)(regs ? xreg(m3[i]) : 3);
            ysrc[i] = (signed char)(regs || part[i] == 2 ? yreg(s) : 3);
            xload[i] = xsrc[i] == 3 && m3[i] != xm;
            if (xload[i]) xm = m3[i];
            yload[i] = ysrc[i] == 3 && (!regs || s != yc);
            if (yload[i]) yc = s;
        }
        // quarter bounds (monotone: the staged y is read in s3 order); a quarter without
        // staged reads collapses onto the previous bound
        int last = 1;  // y[0], y[1] are read from quarter 0 before the first term
        for (int q = 0; q < 4; ++q) {
            qbeg[q] = -1;
            qend[q] = last;
            for (int i = 0; i < COUNT; ++i) {
                const int s = k3[i] - m3[i] + N / 2;
                if (!yload[i] || s / (N / 4) != q) continue;
                if (qbeg[q] < 0) qbeg[q] = i;
                qend[q] = i + 1;
            }
            if (qbeg[q] < 0) qbeg[q] = last;       // no staged read: wait and refill at the same point
            if (q > 0 && qbeg[q] < last) qmono = false;  // a quarter read before the previous one is done
            if (qend[q] < qbeg[q]) qend[q] = qbeg[q];
            last = qend[q];
        }
        qbeg[0] = 0;
    }
    bool qmono = true;
};
// ORDER 1 loads x when the diagonal changes and y per term from the staged row
// in parts 0 and 1 (from registers in part 2); ORDER 2 as the table says.
#ifndef BOLTZ_KCSR_XPF
#define BOLTZ_KCSR_XPF 0  // (removed) x one diagonal ahead: 314 against 305 ms per N=32 RK2 step, spills
#endif
template <int N>
struct KcsrEntry {
    double2 (&acc)[N];
    const double2* X;
    const double2* ys;
    const double2* hs;
    int lane;
    double2 xm, yc, hb, xa, xb, xc, y0, y1, yl;
    template <int I>
    __device__ __forceinline__ void step() {
        constexpr KcsrTab<N> tab{};
        constexpr int k3 = tab.k3[I], m3 = tab.m3[I], s3 = k3 - m3 + N / 2;
        constexpr int xs = tab.xsrc[I], ysr = tab.ysrc[I];
        if constexpr (tab.xload[I]) xm = ldg2(X + (size_t)m3 * kLanes);
        if constexpr (tab.yload[I]) yc = ys[s3 * kLanes + lane];
        if constexpr ((I & 1) == 0) hb = hs[I >> 1];
        const double h = (I & 1) ? hb.y : hb.x;
        const double2 xv = xs == 0 ? xa : xs == 1 ? xb : xs == 2 ? xc : xm;
        const double2 yv = ysr == 0 ? y0 : ysr == 1 ? y1 : ysr == 2 ? yl : yc;
        const double tr = fma(xv.x, yv.x, -xv.y * yv.y);
        const double ti = fma(xv.x, yv.y, xv.y * yv.x);
        acc[k3].x = fma(h, tr, acc[k3].x);
        acc[k3].y = fma(h, ti, acc[k3].y);
    }
};
template <int I, int END>
struct KcsrRun {
    template <typename F>
    __device__ __forceinline__ static void run(F& f) {
        if constexpr (I < END) {
            f.template step<I>();
            KcsrRun<I + 1, END>::run(f);
        }
    }
};
template <int N>
__host__ __device__ constexpr int kcsr_part_begin(int part) {
    int c = 0;
    for (int pt = 0; pt < part; ++pt)
        for (int m = 0; m < N; ++m)
            for (int k = 0; k < N; ++k) c += kcsr_part(N, pt, k, m) ? 1 : 0;
    return c;
}

template <int N>
__global__ void __launch_bounds__(kLanes* kKcsrWarps, BOLTZ_KCSR_MINB)
k_conv_kcsr(const double2* __restrict__ A, double2* __restrict__ B, const double* __restrict__ H,
            const int4* __restrict__ ent, const int* __restrict__ list, int nrows, int ngroups, int lpt_from, int head_lpt) {
    using LY = KcsrLayout<N>;
    constexpr int N3 = N * N * N;
    constexpr unsigned HB = LY::H_BYTES;
    constexpr int P2 = kcsr_part_begin<N>(2);
    [[maybe_unused]] constexpr int PE = KcsrTab<N>::COUNT;
    extern __shared__ __align__(16) char smem[];
    const int2 unit = lpt_unit(list + 3 * nrows + 1, lpt_from, head_lpt);
    const int wi = unit.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int g = unit.y * kKcsrWarps + wid;
    if (g >= ngroups) return;
    const int row = __ldg(list + nrows + 1 + wi);
    const int e0 = __ldg(list + wi), e1 = __ldg(list + wi + 1);
    char* wsm = smem + wid * LY::WARP_BYTES;
    const double2* ys0 = reinterpret_cast<const double2*>(wsm);
    char* xebase = wsm + BOLTZ_KCSR_YBUF * LY::Y_BYTES;
    char* hbase = xebase + BOLTZ_KCSR_YBUF * LY::XE_BYTES;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(hbase + 2 * LY::H_BYTES);
    const double2* Abase = A + (size_t)g * N3 * kLanes;
    const double2* Ag = Abase + lane;
    double2* Brow = B + ((size_t)g * N3 + (size_t)row * N) * kLanes + lane;
    double2 acc[N];
#pragma unroll
    for (int k = 0; k < N; ++k) acc[k] = Brow[(size_t)k * kLanes];  // seeded: every phase-1 row is a pair row
    auto tma_h = [&](int slot, int4 en) {  // the whole warp (converged)
        if constexpr (BOLTZ_TMA_ELECT) {
            bulk_g2s1_elect(bar + slot, hbase + slot * LY::H_BYTES, H + (size_t)(unsigned)en.z, HB);
        } else if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar + slot, HB);
            bulk_g2s(hbase + slot * LY::H_BYTES, H + (size_t)(unsigned)en.z, HB, bar + slot);
        }
    };
    auto tma_y = [&](int slot, int4 en) {  // the whole warp (converged)
        double2* yd = const_cast<double2*>(ys0) + (BOLTZ_KCSR_YBUF == 2 ? slot * N * kLanes : 0);
        if constexpr (BOLTZ_TMA_ELECT && LY::XE_BYTES > 0) {
            char* xe = xebase + slot * LY::XE_BYTES;
            bulk_g2s3_elect(bar + slot, yd, Abase + (size_t)en.y * kLanes, LY::Y_BYTES, xe,
                            Abase + (size_t)en.x * kLanes, 2 * kLanes * 16, xe + 2 * kLanes * 16,
                            Abase + (size_t)(en.x + N - 1) * kLanes, kLanes * 16);
        } else if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(bar + slot, LY::Y_BYTES + LY::XE_BYTES);
            bulk_g2s(yd, Abase + (size_t)en.y * kLanes, LY::Y_BYTES, bar + slot);
            if constexpr (LY::XE_BYTES > 0) {
                char* xe = xebase + slot * LY::XE_BYTES;
                bulk_g2s(xe, Abase + (size_t)en.x * kLanes, 2 * kLanes * 16, bar + slot);
                bulk_g2s(xe + 2 * kLanes * 16, Abase + (size_t)(en.x + N - 1) * kLanes, kLanes * 16, bar + slot);
            }
        }
    };
    EntWin win(ent, e0, e1, lane);
    auto entry = [&](int e) { return win.get(e); };
    if (e0 < e1) {
        if (lane == 0) {
            mbar_init(bar, 2);
            mbar_init(bar + 1, 2);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        int4 en = entry(e0);
        tma_y(0, en);
        tma_h(0, en);
        mbar_wait(bar, 0);
        for (int e = e0; e < e1; ++e) {
            const int i = e - e0, cur = i & 1;
            const bool more = e + 1 < e1;
            const int4 nx = more ? entry(e + 1) : en;
            __syncwarp();  // every lane finished reading H[cur^1] (and y[cur^1])
            if (more) tma_h(cur ^ 1, nx);
            const double2* ys = ys0 + (BOLTZ_KCSR_YBUF == 2 ? cur * N * kLanes : 0);
            if (BOLTZ_KCSR_YBUF == 2 && more) tma_y(cur ^ 1, nx);
            KcsrEntry<N> f{acc, Ag + (size_t)en.x * kLanes, ys,
                           reinterpret_cast<const double2*>(hbase + cur * LY::H_BYTES), lane};
            if constexpr (LY::XE_BYTES > 0) {
                const double2* xe = reinterpret_cast<const double2*>(xebase + cur * LY::XE_BYTES);
                f.xa = xe[lane];
                f.xb = xe[kLanes + lane];
                f.xc = xe[2 * kLanes + lane];
                f.y0 = ys[lane];
                f.y1 = ys[kLanes + lane];
                f.yl = ys[(N - 1) * kLanes + lane];
            }
            KcsrRun<0, P2>::run(f);  // parts 0 and 1: y from the staged row
            if constexpr (BOLTZ_KCSR_YBUF == 1 || BOLTZ_KCSR_YREG) {
                f.y0 = ys[lane];
                f.y1 = ys[kLanes + lane];
                f.yl = ys[(N - 1) * kLanes + lane];
                if constexpr (BOLTZ_KCSR_YBUF == 1) {
                    __syncwarp();  // every lane read the y row: the buffer may be refilled
                    if (more) tma_y(cur ^ 1, nx);
                }
                KcsrRun<P2, PE>::run(f);  // part 2: y[0], y[1], y[N-1] in registers
            }
            if (more) mbar_wait(bar + (cur ^ 1), (unsigned)(((i + 1) >> 1) & 1));
            en = nx;
        }
    }
#pragma unroll
    for (int k = 0; k < N; ++k) Brow[(size_t)k * kLanes] = acc[k];  // raw: phase 2 continues the row
}

// ---------------------------------------------------------------------------
// k_conv_kcsrq (BOLTZ_KCSR_YBUF 4): k_conv_kcsr with ONE y row per warp,
// refilled by quarters.  The s3-grouped term order reads the staged y in s3
// order, so quarter q of the next entry's y row is issued as soon as the
// current entry has read its quarter q (KcsrTab qend), a whole entry ahead of
// its use; the edge rows x[0], x[1], x[N-1] and y[N-1] (read from the start)
// ride with the H slab in a double-buffered slot.  22.3 KB per warp instead of
// 37.6 KB: 8 warps per SM (register-bound) instead of 6 (shared-memory-bound).
// Measured on B200 (cfg5-shaped collide, 2048 cells, two runs): 145.0 / 145.6
// against 144.9 / 144.9 ms with k_conv_kcsr -- the extra warps buy nothing, so
// the REST launch is bound by L2 throughput (67%), not by latency; opt-in
// (BOLTZ_KCSR_YBUF=4), oracle parity and the checksum as k_conv_kcsr.
// ---------------------------------------------------------------------------
template <int N>
struct KcsrqLayout {
    static constexpr int Y_BYTES = N * kLanes * 16;  // one y row
    static constexpr int Q_BYTES = Y_BYTES / 4;
    static constexpr int XE_BYTES = 4 * kLanes * 16;  // x[0], x[1], x[N-1], y[N-1]
    static constexpr int H_BYTES = (kcsr_slab(N) * 8 + 15) / 16 * 16;
    static constexpr int SLOT_BYTES = XE_BYTES + H_BYTES;
    static constexpr int WARP_BYTES = Y_BYTES + 2 * SLOT_BYTES + 6 * 8;  // + 2 slot and 4 quarter mbarriers
};
#ifndef BOLTZ_KCSRQ_MINB
#define BOLTZ_KCSRQ_MINB 4
#endif
template <int N>
__global__ void __launch_bounds__(kLanes* kKcsrWarps, BOLTZ_KCSRQ_MINB)
k_conv_kcsrq(const double2* __restrict__ A, double2* __restrict__ B, const double* __restrict__ H,
             const int4* __restrict__ ent, const int* __restrict__ list, int nrows, int ngroups, int lpt_from,
             int head_lpt) {
    using LY = KcsrqLayout<N>;
    constexpr KcsrTab<N> tab{};
    static_assert(tab.qmono, "k_conv_kcsrq: the staged y must be read in quarter order");
    constexpr int PE = KcsrTab<N>::COUNT;
    constexpr int QB1 = tab.qbeg[1], QB2 = tab.qbeg[2], QB3 = tab.qbeg[3];
    constexpr int QE0 = tab.qend[0], QE1 = tab.qend[1], QE2 = tab.qend[2], QE3 = tab.qend[3];
    constexpr int N3 = N * N * N, QS = N / 4;
    constexpr unsigned HB = kcsr_slab(N) * 8;
    extern __shared__ __align__(16) char smem[];
    const int2 unit = lpt_unit(list + 3 * nrows + 1, lpt_from, head_lpt);
    const int wi = unit.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int g = unit.y * kKcsrWarps + wid;
    if (g >= ngroups) return;
    const int row = __ldg(list + nrows + 1 + wi);
    const int e0 = __ldg(list + wi), e1 = __ldg(list + wi + 1);
    char* wsm = smem + wid * LY::WARP_BYTES;
    double2* ys = reinterpret_cast<double2*>(wsm);
    char* slots = wsm + LY::Y_BYTES;
    unsigned long long* barE = reinterpret_cast<unsigned long long*>(slots + 2 * LY::SLOT_BYTES);
    unsigned long long* barQ = barE + 2;
    const double2* Abase = A + (size_t)g * N3 * kLanes;
    const double2* Ag = Abase + lane;
    double2* Brow = B + ((size_t)g * N3 + (size_t)row * N) * kLanes + lane;
    double2 acc[N];
#pragma unroll
    for (int k = 0; k < N; ++k) acc[k] = Brow[(size_t)k * kLanes];  // seeded: every REST row is a pair row
    auto tma_slot = [&](int slot, int4 en) {  // the edge rows + the H slab of entry en
        if (lane == 0) {
            char* sl = slots + slot * LY::SLOT_BYTES;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(barE + slot, LY::XE_BYTES + HB);
            bulk_g2s(sl, Abase + (size_t)en.x * kLanes, 2 * kLanes * 16, barE + slot);
            bulk_g2s(sl + 2 * kLanes * 16, Abase + (size_t)(en.x + N - 1) * kLanes, kLanes * 16, barE + slot);
            bulk_g2s(sl + 3 * kLanes * 16, Abase + (size_t)(en.y + N - 1) * kLanes, kLanes * 16, barE + slot);
            bulk_g2s(sl + LY::XE_BYTES, H + (size_t)(unsigned)en.z, HB, barE + slot);
        }
    };
    auto tma_q = [&](int q, int4 en) {  // quarter q of entry en's y row
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(barQ + q, LY::Q_BYTES);
            bulk_g2s(ys + q * QS * kLanes, Abase + (size_t)(en.y + q * QS) * kLanes, LY::Q_BYTES, barQ + q);
        }
    };
    EntWin win(ent, e0, e1, lane);
    if (e0 < e1) {
        if (lane == 0) {
            for (int b = 0; b < 6; ++b) mbar_init(barE + b, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        int4 en = win.get(e0);
        tma_slot(0, en);
        for (int q = 0; q < 4; ++q) tma_q(q, en);
        mbar_wait(barE, 0);
        for (int e = e0; e < e1; ++e) {
            const int i = e - e0, cur = i & 1;
            const unsigned qp = (unsigned)(i & 1);  // each quarter barrier completes once per entry
            const bool more = e + 1 < e1;
            const int4 nx = more ? win.get(e + 1) : en;
            __syncwarp();  // every lane finished with slot cur^1 (entry i-1)
            if (more) tma_slot(cur ^ 1, nx);
            const double2* xe = reinterpret_cast<const double2*>(slots + cur * LY::SLOT_BYTES);
            KcsrEntry<N> f{acc, Ag + (size_t)en.x * kLanes, ys,
                           reinterpret_cast<const double2*>(slots + cur * LY::SLOT_BYTES + LY::XE_BYTES), lane};
            f.xa = xe[lane];
            f.xb = xe[kLanes + lane];
            f.xc = xe[2 * kLanes + lane];
            f.yl = xe[3 * kLanes + lane];
            mbar_wait(barQ, qp);
            f.y0 = ys[lane];
            f.y1 = ys[kLanes + lane];
            auto refill = [&](int q) {
                __syncwarp();  // every lane has read quarter q of this entry's y
                if (more) tma_q(q, nx);
            };
            KcsrRun<0, QE0>::run(f);
            refill(0);
            KcsrRun<QE0, QB1>::run(f);
            mbar_wait(barQ + 1, qp);
            KcsrRun<QB1, QE1>::run(f);
            refill(1);
            KcsrRun<QE1, QB2>::run(f);
            mbar_wait(barQ + 2, qp);
            KcsrRun<QB2, QE2>::run(f);
            refill(2);
            KcsrRun<QE2, QB3>::run(f);
            mbar_wait(barQ + 3, qp);
            KcsrRun<QB3, QE3>::run(f);
            refill(3);
            KcsrRun<QE3, PE>::run(f);
            if (more) mbar_wait(barE + (cur ^ 1), (unsigned)(((i + 1) >> 1) & 1));
            en = nx;
        }
    }
#pragma unroll
    for (int k = 0; k < N; ++k) Brow[(size_t)k * kLanes] = acc[k];  // raw: phase 2 continues the row
}

// ---- H table builder.  Entry e = output row (k1,k2) x representative input
// row (m1,m2) (entk = {k1,k2,m1,m2}) with meta[e] = {H offset, band type};
// term[ts.off[type] + pos] = (k3, m3) of slab position pos, or (-1,-1) for
// padding.  Folding: H = G'(k,m) + G'(k,sigma m), G' = G omega_m,
// omega_m = c3(m) dzeta^3 (velocity_grid.hpp:43-46); the self-paired input
// row keeps its m3 <= s3 half.
struct TermSet {
    const short2* term;
    int off[kBandTypes];
    int slab[kBandTypes];
    int slab_max;
};

template <typename GF>
__device__ __forceinline__ double folded_h(int n, double w3, int4 q, short2 km, GF&& G) {
    const int h = n / 2;
    const int k2 = q.y, m1 = q.z, m2 = q.w, k3 = km.x, m3 = km.y;
    const int s1 = q.x - m1 + h, s2 = k2 - m2 + h, s3 = k3 - m3 + h;
    const double wm = axis_coeff(n, m1) * axis_coeff(n, m2) * axis_coeff(n, m3) * w3;
    const double ws = axis_coeff(n, s1) * axis_coeff(n, s2) * axis_coeff(n, s3) * w3;
    const bool self_row = (m1 == s1) && (m2 == s2);
    if (!self_row || m3 < s3) return G(k3, m1, m2, m3) * wm + G(k3, s1, s2, s3) * ws;
    if (m3 == s3) return G(k3, m1, m2, m3) * wm;
    return 0.0;
}

// from one k1-plane of the caller's dense zeta-major G:
// Gk1[(k2*N + k3) * N^3 + m]; list[e_begin..e_end) = the entries of that plane
// mode 0: the entries' own terms (plane k1 = q.x); mode 1: only their
// partner-row terms (term.x >= kMirrorTermFlag, plane N - q.x), which must not
// be touched in mode 0
__global__ void k_build_H(const double* __restrict__ Gk1, double* __restrict__ H, const int4* __restrict__ entk,
                          const int2* __restrict__ meta, const int* __restrict__ list, int e_begin, int e_end,
                          TermSet ts, int n, double w3, int mode) {
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= (long long)(e_end - e_begin) * ts.slab_max) return;
    const int e = list[e_begin + (int)(tid / ts.slab_max)];
    const int pos = (int)(tid % ts.slab_max);
    const int2 mt = meta[e];
    if (pos >= ts.slab[mt.y]) return;
    int4 q = entk[e];
    short2 km = ts.term[ts.off[mt.y] + pos];
    const bool partner = km.x >= kMirrorTermFlag;
    if (partner != (mode == 1)) return;
    if (partner) {
        km.x -= kMirrorTermFlag;
        q = mirror_q(n, q);
    }
    double out = 0.0;
    if (km.x >= 0) {
        const long long n3 = (long long)n * n * n;
        out = folded_h(n, w3, q, km, [&](int k3, int a1, int a2, int a3) {
            return Gk1[((long long)q.y * n + k3) * n3 + ((long long)a1 * n + a2) * n + a3];
        });
    }
    H[(size_t)(unsigned)mt.x + pos] = out;
}

}  // namespace boltz_gpu
