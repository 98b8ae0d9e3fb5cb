// line.cuh -- K1 / K3 with one FFT line per thread (N = 8, 16).  The first axis
// pass runs from the loaded data into registers and the last one from registers
// to the output, so a transform costs two shared-memory round trips instead of
// the staged kernels' four (fused.cuh, which remains for N = 12, 24).
//
//   k_fwd_line_tma:    user f [cell][N^3]  -> group fhat      (fourier.hpp:11-12)
//   k_inv_line2<FWD>:  group s_k*Qhat       -> out = base + coef * P_N(Re iFFT)
//                      (+ max|Im|; inverse fourier.hpp:15-17, projection
//                      SPEC.md:204-212, RK2 axpy SPEC.md:383-391); FWD: the
//                      RK2 stage value goes straight on to its forward
//                      transform into A_next, never touching HBM
// Both move every HBM byte by TMA (2D tensor maps built per call on the host:
// make_group_tmap, make_cells_tmap in boltz_cuda.cu).  k_fwd_line / k_inv_line
// are the same transforms with per-lane loads and stores (BOLTZ_LINE_TMA=0,
// BOLTZ_LINE_INV2=0, and user arrays that are not 16-byte aligned).
//
// Thread t of the N^2 threads owns the lines (a, b) = (t / N, t % N) of every
// pass: along i3 at (i1, i2) = (a, b), along i2 at (i1, i3) = (a, b), along i1 at
// (i2, i3) = (a, b).  Moments are summed per thread over the last pass's axis and
// reduced in a fixed order (a shuffle tree per 16 consecutive lines, then the
// 16-line partials in line order): deterministic, independent of the batch and
// of the cells-per-CTA variant.  Cells past ncells (the group's padding lanes)
// read as zero.  HBM traffic per cell (N = 16): K1 32 KiB in + 64 KiB out;
// K3 64 KiB + 32 KiB base in, 32 KiB (or, FWD, 64 KiB fhat) out.
#pragma once
#include <cuda.h>  // CUtensorMap (the group-layout stores of BOLTZ_LINE_TMA)
#include "common.cuh"
#include "fft.cuh"

namespace boltz_gpu {

// the line kernels' TMA plane loads / stores issued by every warp's elected
// lane (2 planes per warp at N = 16) instead of one thread issuing all of them.
// B200, cfg2 RK2 step (three runs): K3 (k_inv_line2, both launches) 0.360 ->
// 0.350 ms; K1's per-block plane stores lost (0.107 -> 0.114 ms), so K1 keeps
// thread 0 (BOLTZ_LINE_SPREAD_K1)
#ifndef BOLTZ_LINE_SPREAD
#define BOLTZ_LINE_SPREAD 1
#endif
#ifndef BOLTZ_LINE_SPREAD_K1
#define BOLTZ_LINE_SPREAD_K1 0
#endif
// K1's plane stores from warp 0 with the predicate inside the asm (elect.sync
// picks lane 0 of the converged warp: thread 0, which waits on the bulk group);
// measured slower too (K1 0.108 -> 0.114 ms), off
#ifndef BOLTZ_LINE_K1_ELECT
#define BOLTZ_LINE_K1_ELECT 0
#endif
#ifndef BOLTZ_LINE_MINB
#define BOLTZ_LINE_MINB 2  // CTAs per SM the line kernels are compiled for (registers), one cell per CTA
#endif
// cells per CTA: 1, or 2 adjacent cells of a group handled by the two half-warps
// of every warp (lanes 0-15 and 16-31 take the same 16 lines of the two cells),
// so that each group-layout access is a whole 32-byte sector (two 16-byte
// lanes) instead of half of one
// (the launcher picks: 2 for device-memory calls -- cfg2 RK2 step K1 0.182 ->
// 0.168 ms, K3 0.523 -> 0.497 ms -- and 1 inside the two-stream host pipeline,
// where the 141 KB two-cell CTA would keep the other stream's K2 off the SM:
// e2e 657k against 661-670k evals/s with it)
template <int N, int CPB_ = 1>
struct Line {
    static constexpr int N3 = N * N * N;
    static constexpr int CPB = CPB_;
    static constexpr int THREADS = N * N * CPB;
    static constexpr int WARPS = (THREADS + 31) / 32;
    static constexpr int ROW = N + 1;  // padded rows: the three passes are bank-conflict free
    static constexpr int CELL = N * N * ROW;
    static constexpr int HW = N * N / 16;  // 16-line groups per cell (the moments' reduction units)
    static constexpr int SMEM = CPB * CELL * 16 + CPB * HW * 6 * 8 + CPB * 8 * 8;  // cubes + reduction + lambda
    __device__ static int at(int i1, int i2, int i3) { return (i1 * N + i2) * ROW + i3; }
    // thread t -> (cell of the CTA, line): with 2 cells the half-warps split by cell
    __device__ static int sub(int t) { return CPB == 2 ? (t >> 4) & 1 : 0; }
    __device__ static int line(int t) { return CPB == 2 ? ((t >> 5) << 4) | (t & 15) : t; }
    static constexpr unsigned MINB = CPB == 2 ? 1 : BOLTZ_LINE_MINB;
};
// the line kernels serve these N (N^2 a multiple of 32: whole warps in the shuffle reduction)
__host__ __device__ constexpr bool line_n(int n) { return n == 8 || n == 16; }

// one in-smem pass along axis 1 (i2) of the lines (i1, i3) = (a, b)
template <int N, int SIGN>
__device__ __forceinline__ void line_pass_axis1(double2* sm, int a, int b) {
    using LN = Line<N>;
    double2 x[N];
#pragma unroll
    for (int j = 0; j < N; ++j) x[j] = sm[LN::at(a, j, b)];
    RegFFT<N, SIGN, N>::run(x);
#pragma unroll
    for (int j = 0; j < N; ++j) sm[LN::at(a, j, b)] = x[j];
}

// BOLTZ_LINE_PERSIST: K1 runs a grid-stride loop over its blocks of CPB cells
// (grid = the resident CTAs), loading the next block's lines while the current
// one is in passes 2 and 3
#ifndef BOLTZ_LINE_PERSIST
#define BOLTZ_LINE_PERSIST 1
#endif
// blocks = cells / CPB (the groups' padding lanes included); block = CPB N^2 threads
template <int N, int CPB>
__global__ void __launch_bounds__(Line<N, CPB>::THREADS, Line<N, CPB>::MINB)
k_fwd_line(const double* __restrict__ f, double2* __restrict__ A, long long ncells, double scale,
           int* __restrict__ flag) {
    using LN = Line<N, CPB>;
    constexpr int N3 = LN::N3;
    extern __shared__ __align__(16) double2 smem_line[];
    const int t = threadIdx.x, sub = LN::sub(t), ln = LN::line(t), a = ln / N, b = ln % N;
    double2* sm = smem_line + sub * LN::CELL;
    const long long nblk = (ncells + kLanes - 1) / kLanes * kLanes / CPB;
    const long long stride = BOLTZ_LINE_PERSIST ? gridDim.x : nblk;
    const double cab = axis_coeff(N, a) * axis_coeff(N, b);
    // pass 1 (axis 2, i3) from global: the line (a, b, :) is N contiguous doubles,
    // loaded as N / 2 16-byte loads (f is 16-byte aligned: the callers check)
    double fv[N];
    auto load = [&](long long blk) {
        const long long cell = blk * CPB + sub;
        const bool live = blk < nblk && cell < ncells;
        const double2* fl = reinterpret_cast<const double2*>(f + (size_t)cell * N3 + (size_t)(a * N + b) * N);
#pragma unroll
        for (int j = 0; j < N / 2; ++j) {
            const double2 u = live ? ldg2(fl + j) : make_double2(0.0, 0.0);
            fv[2 * j] = u.x;
            fv[2 * j + 1] = u.y;
        }
    };
    load(blockIdx.x);
    for (long long blk = blockIdx.x; blk < nblk; blk += stride) {
        const long long cell = blk * CPB + sub;
        double2 x[N];
        bool bad = false;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const double v = fv[j];
            bad |= !isfinite(v);
            double w = cab * axis_coeff(N, j);  // s_m c_m (fourier.hpp:19-22)
            if ((a + b + j) & 1) w = -w;
            x[j] = make_double2(v * w, 0.0);
        }
        if (bad) atomicOr(flag, 1);
        if (BOLTZ_LINE_PERSIST) load(blk + stride);  // in flight through passes 2 and 3
        RegFFT<N, -1, N>::run(x);
#pragma unroll
        for (int j = 0; j < N; ++j) sm[LN::at(a, b, j)] = x[j];
        __syncthreads();
        line_pass_axis1<N, -1>(sm, a, b);
        __syncthreads();
        // pass 3 (axis 0, i1) to global: scale * par * s_k into the group layout
#pragma unroll
        for (int j = 0; j < N; ++j) x[j] = sm[LN::at(j, a, b)];
        RegFFT<N, -1, N>::run(x);
        const long long g = cell / kLanes;
        const int lane = (int)(cell % kLanes);
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const double s = ((j + a + b) & 1) ? -scale : scale;
            A[((size_t)g * N3 + (size_t)(j * N + a) * N + b) * kLanes + lane] = make_double2(x[j].x * s, x[j].y * s);
        }
        if (BOLTZ_LINE_PERSIST) __syncthreads();  // every pass-3 read done before the next pass 1 writes
    }
}

// BOLTZ_LINE_TMA: the group-layout output of a line kernel leaves through
// shared memory by 2D TMA tensor stores (one per i1 plane) instead of 16-byte
// per-lane stores, each of which touches N^2 / 16 separate 128-byte lines
#ifndef BOLTZ_LINE_TMA
#define BOLTZ_LINE_TMA 1
#endif
// the group array X[g][idx][lane] as a 2D tensor of doubles: {2 kLanes, groups N^3}
// (host: make_group_tmap); one box = one i1 plane of CPB adjacent cells
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                 ::"l"(map), "r"(c0), "r"(c1), "r"(smem_u32(src)) : "memory");
}
// the same copies issued by one elected lane of a converged warp (the predicate
// inside the asm: no divergent single-thread region around the TMA instruction)
__device__ __forceinline__ void tma_store_2d_elect(const CUtensorMap* map, const void* src, int c0, int c1) {
    asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n"
                 " @p cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n}"
                 ::"l"(map), "r"(c0), "r"(c1), "r"(smem_u32(src)) : "memory");
}
__device__ __forceinline__ void bulk_commit_elect() {
    asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n @p cp.async.bulk.commit_group;\n}" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_elect() {
    asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n @p cp.async.bulk.wait_group.read 0;\n}" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all_elect() {
    asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n @p cp.async.bulk.wait_group 0;\n}" ::: "memory");
}
__device__ __forceinline__ void bulk_commit_wait_all_elect() {
    asm volatile("{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n"
                 " @p cp.async.bulk.commit_group;\n @p cp.async.bulk.wait_group 0;\n}" ::: "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// a user array [cell][N^3] as a 2D TMA tensor of doubles {N, cells N^2}: row =
// one line (a, b, :) of N doubles, box = one cell (N^2 rows), landed with the
// 128-byte (N = 16) or 64-byte (N = 8) swizzle so that lanes reading chunk c of
// consecutive lines hit distinct banks (host: make_cells_tmap)
template <int N>
__device__ __forceinline__ int swz(int byte) {
    constexpr int mask = N * 8 >= 128 ? 7 : N * 8 >= 64 ? 3 : 1;
    return byte ^ (((byte >> 7) & mask) << 4);
}
__device__ __forceinline__ void tma_load_2d_elect(void* dst, const CUtensorMap* map, int c0, int c1,
                                                  unsigned long long* bar) {
    asm volatile(
        "{\n .reg .pred p;\n elect.sync _|p, 0xffffffff;\n"
        " @p cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n}"
        ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)) : "memory");
}
// BOLTZ_LINE_TMA_LOAD: K1 also takes f by TMA (swizzled, one box per cell), the
// next block's box issued as soon as the current one is in registers
#ifndef BOLTZ_LINE_TMA_LOAD
#define BOLTZ_LINE_TMA_LOAD 1
#endif
#ifndef BOLTZ_LINE_WAR_FENCE
#define BOLTZ_LINE_WAR_FENCE 1
#endif
template <int N, int CPB>
struct LineTma {
    static constexpr int F_BYTES = CPB * N * N * N * 8;             // the f image (swizzled lines)
    static constexpr int SMEM = Line<N, CPB>::SMEM + (BOLTZ_LINE_TMA_LOAD ? F_BYTES + 1024 + 16 : 0);
};

// K1 with the output by TMA (grid-stride over blocks of CPB cells, as k_fwd_line).
// After pass 3 the block's values go to a dense staging image of its group
// rows -- plane j (idx j N^2 .. j N^2 + N^2 - 1) x CPB cells, 16 bytes each --
// over the cube, and thread 0 stores the N planes; the next block waits for
// those reads before it rewrites the cube.
template <int N, int CPB>
__global__ void __launch_bounds__(Line<N, CPB>::THREADS, Line<N, CPB>::MINB)
k_fwd_line_tma(const double* __restrict__ f, const __grid_constant__ CUtensorMap tmF,
               const __grid_constant__ CUtensorMap tmA, long long ncells, double scale, int* __restrict__ flag) {
    using LN = Line<N, CPB>;
    constexpr int N3 = LN::N3, NN = N * N;
    static_assert(N3 * CPB <= CPB * LN::CELL, "the staging image fits over the cubes");
    extern __shared__ __align__(128) double2 smem_line_tma[];  // TMA: 128-byte aligned
    double2* smem_line = smem_line_tma;
    const int t = threadIdx.x, sub = LN::sub(t), ln = LN::line(t), a = ln / N, b = ln % N;
    double2* sm = smem_line + sub * LN::CELL;
    const long long nblk = (ncells + kLanes - 1) / kLanes * kLanes / CPB;
    const double cab = axis_coeff(N, a) * axis_coeff(N, b);
    double fv[N];
    // the f image: after the cubes, 1024-byte aligned (the swizzle atom)
    char* fimg = reinterpret_cast<char*>(smem_line + CPB * LN::CELL);
    fimg += (1024 - (smem_u32(fimg) & 1023)) & 1023;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(fimg + LineTma<N, CPB>::F_BYTES);
    unsigned phase = 0;
    auto issue = [&](long long blk) {  // thread 0: the CPB cells of block blk (rows past the tensor read as 0)
        if (blk >= nblk) return;
        mbar_expect_tx(bar, LineTma<N, CPB>::F_BYTES);
#pragma unroll
        for (int c = 0; c < CPB; ++c) tma_load_2d(fimg + c * N3 * 8, &tmF, 0, (int)((blk * CPB + c) * NN), bar);
    };
    auto load = [&](long long blk) {
        if constexpr (BOLTZ_LINE_TMA_LOAD) {
            mbar_wait(bar, phase);
            phase ^= 1;
            const char* line = fimg + sub * N3 * 8;
#pragma unroll
            for (int j = 0; j < N / 2; ++j) {
                const double2 u = *reinterpret_cast<const double2*>(line + swz<N>(ln * N * 8 + j * 16));
                fv[2 * j] = u.x;
                fv[2 * j + 1] = u.y;
            }
        } else {
            const long long cell = blk * CPB + sub;
            const bool live = blk < nblk && cell < ncells;
            const double2* fl = reinterpret_cast<const double2*>(f + (size_t)cell * N3 + (size_t)(a * N + b) * N);
#pragma unroll
            for (int j = 0; j < N / 2; ++j) {
                const double2 u = live ? ldg2(fl + j) : make_double2(0.0, 0.0);
                fv[2 * j] = u.x;
                fv[2 * j + 1] = u.y;
            }
        }
    };
    if constexpr (BOLTZ_LINE_TMA_LOAD) {
        if (t == 0) {
            mbar_init(bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (t == 0) issue(blockIdx.x);
        load(blockIdx.x);
        if (BOLTZ_LINE_WAR_FENCE) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();  // every thread holds its lines: the image may be refilled
        if (t == 0) issue(blockIdx.x + gridDim.x);
    } else {
        load(blockIdx.x);
    }
    for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
        double2 x[N];
        bool bad = false;
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const double v = fv[j];
            bad |= !isfinite(v);
            double w = cab * axis_coeff(N, j);  // s_m c_m (fourier.hpp:19-22)
            if ((a + b + j) & 1) w = -w;
            x[j] = make_double2(v * w, 0.0);
        }
        if (bad) atomicOr(flag, 1);
        if constexpr (!BOLTZ_LINE_TMA_LOAD) load(blk + gridDim.x);  // in flight through passes 2 and 3
        RegFFT<N, -1, N>::run(x);
        if (blk != blockIdx.x) {  // the previous block's stores have read the staging image
            if constexpr (BOLTZ_LINE_SPREAD_K1) bulk_wait_read_elect();  // every warp's own stores
            else if (t == 0) bulk_wait_read();
            __syncthreads();
        }
#pragma unroll
        for (int j = 0; j < N; ++j) sm[LN::at(a, b, j)] = x[j];
        __syncthreads();
        line_pass_axis1<N, -1>(sm, a, b);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < N; ++j) x[j] = sm[LN::at(j, a, b)];
        RegFFT<N, -1, N>::run(x);
        __syncthreads();  // every pass-3 read done: the cubes become the staging image
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const double s = ((j + a + b) & 1) ? -scale : scale;
            smem_line[(j * NN + ln) * CPB + sub] = make_double2(x[j].x * s, x[j].y * s);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if constexpr (BOLTZ_LINE_TMA_LOAD) {
            if (blk + gridDim.x < nblk) load(blk + gridDim.x);  // the next block's lines (landed meanwhile)
            if (BOLTZ_LINE_WAR_FENCE) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        __syncthreads();
        if constexpr (BOLTZ_LINE_SPREAD_K1) {  // each warp's elected lane stores its planes
            const long long cell0 = blk * CPB;
            const int c0 = (int)(cell0 % kLanes) * 2, row0 = (int)(cell0 / kLanes) * N3;
            for (int j = t >> 5; j < N; j += LN::WARPS) tma_store_2d_elect(&tmA, smem_line + j * NN * CPB, c0, row0 + j * NN);
            bulk_commit_elect();
            if constexpr (BOLTZ_LINE_TMA_LOAD)
                if (t == 0) issue(blk + 2 * (long long)gridDim.x);
        } else if (BOLTZ_LINE_K1_ELECT && t < 32) {  // warp 0, the stores by its elected lane (= thread 0)
            const long long cell0 = blk * CPB;
            const int c0 = (int)(cell0 % kLanes) * 2, row0 = (int)(cell0 / kLanes) * N3;
#pragma unroll
            for (int j = 0; j < N; ++j) tma_store_2d_elect(&tmA, smem_line + j * NN * CPB, c0, row0 + j * NN);
            bulk_commit_elect();
            if constexpr (BOLTZ_LINE_TMA_LOAD)
                if (t == 0) issue(blk + 2 * (long long)gridDim.x);
        } else if (!BOLTZ_LINE_K1_ELECT && t == 0) {
            const long long cell0 = blk * CPB;
            const int c0 = (int)(cell0 % kLanes) * 2, row0 = (int)(cell0 / kLanes) * N3;
#pragma unroll 1
            for (int j = 0; j < N; ++j) tma_store_2d(&tmA, smem_line + j * NN * CPB, c0, row0 + j * NN);
            bulk_commit();
            if constexpr (BOLTZ_LINE_TMA_LOAD) issue(blk + 2 * (long long)gridDim.x);
        }
    }
    if constexpr (BOLTZ_LINE_SPREAD_K1) bulk_wait_all_elect();
    else if (t == 0) bulk_wait_all();
}

template <int N, bool FWD, int CPB>
__global__ void __launch_bounds__(Line<N, CPB>::THREADS, Line<N, CPB>::MINB)
k_inv_line(const double2* __restrict__ B, const double* __restrict__ base, double* __restrict__ out,
           double* __restrict__ maximag, long long ncells, double scale, double coef, ProjConst pc,
           int* __restrict__ flag, double2* __restrict__ A_next, const __grid_constant__ CUtensorMap tmNext,
           double fwd_scale) {
    using LN = Line<N, CPB>;
    constexpr int N3 = LN::N3, NN = N * N;
    extern __shared__ __align__(128) double2 smem_line_tma[];  // TMA (FWD): 128-byte aligned
    double2* smem_line = smem_line_tma;
    double* red = reinterpret_cast<double*>(smem_line + CPB * LN::CELL);  // [CPB][HW][6]
    double* lam = red + CPB * LN::HW * 6;                                // [CPB][8]
    const int t = threadIdx.x, sub = LN::sub(t), ln = LN::line(t), a = ln / N, b = ln % N;
    double2* sm = smem_line + sub * LN::CELL;
    const long long cell = (long long)blockIdx.x * CPB + sub;
    const bool live = cell < ncells;
    const long long g = cell / kLanes;
    const int lane = (int)(cell % kLanes);
    // the RK2 base this thread applies at the end, prefetched now: FWD -- the
    // line (a, b, :), contiguous; otherwise nodes ln + k N^2 (coalesced)
    double bv[N];
    if constexpr (FWD) {  // N / 2 16-byte loads (base is 16-byte aligned: the callers check)
        const double2* bl = reinterpret_cast<const double2*>(base + (size_t)cell * N3 + (size_t)(a * N + b) * N);
#pragma unroll
        for (int j = 0; j < N / 2; ++j) {
            const double2 u = (live && base) ? ldg2(bl + j) : make_double2(0.0, 0.0);
            bv[2 * j] = u.x;
            bv[2 * j + 1] = u.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < N; ++j)
            bv[j] = (live && base) ? __ldg(base + (size_t)cell * N3 + (size_t)j * NN + ln) : 0.0;
    }
    // pass 1 (axis 2, i3) from the group layout
    double2 x[N];
#pragma unroll
    for (int j = 0; j < N; ++j)
        x[j] = live ? ldg2(B + ((size_t)g * N3 + (size_t)(a * N + b) * N + j) * kLanes + lane) : make_double2(0.0, 0.0);
    RegFFT<N, +1, N>::run(x);
#pragma unroll
    for (int j = 0; j < N; ++j) sm[LN::at(a, b, j)] = x[j];
    __syncthreads();
    line_pass_axis1<N, +1>(sm, a, b);
    __syncthreads();
    // pass 3 (axis 0, i1) in registers: Qt = Re(scale * par * s_k * z), its
    // moments over i1 and max|Im| (the thread's (i2, i3) = (a, b) are fixed)
#pragma unroll
    for (int j = 0; j < N; ++j) x[j] = sm[LN::at(j, a, b)];
    RegFFT<N, +1, N>::run(x);
    const double dv3 = pc.dv * pc.dv * pc.dv;
    const double fv2 = pc.dv * (a - N / 2), fv3 = pc.dv * (b - N / 2);
    const double fw23 = axis_coeff(N, a) * axis_coeff(N, b) * dv3;
    const double sg23 = ((a + b) & 1) ? -scale : scale;
    double s0 = 0.0, s1 = 0.0, s4 = 0.0, mi = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const double q = x[j].x * ((j & 1) ? -sg23 : sg23);
        sm[LN::at(j, a, b)].x = q;
        const double v1 = pc.dv * (j - N / 2);
        const double cq = axis_coeff(N, j) * q;
        s0 += cq;
        s1 = fma(v1, cq, s1);
        s4 = fma(v1 * v1, cq, s4);
        mi = fmax(mi, fabs(x[j].y));
    }
    double part[6];
    part[0] = fw23 * s0;
    part[1] = fw23 * s1;
    part[2] = fv2 * part[0];
    part[3] = fv3 * part[0];
    part[4] = fw23 * fma(fv2 * fv2 + fv3 * fv3, s0, s4);
    part[5] = mi * fabs(scale);
    // shuffle tree over each half-warp (16 consecutive lines of one cell), then
    // the 16-line partials in line order: the same arithmetic for 1 and 2 cells
    // per CTA, so both variants give bitwise the same cell
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        double v = part[k];
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            const double u = __shfl_xor_sync(0xffffffffu, v, o);
            v = (k == 5) ? fmax(v, u) : v + u;
        }
        if ((ln & 15) == 0) red[(sub * LN::HW + (ln >> 4)) * 6 + k] = v;
    }
    __syncthreads();
    if (t < CPB) {
        const int c = t;
        const long long cl = (long long)blockIdx.x * CPB + c;
        double m[6] = {0, 0, 0, 0, 0, 0};
        for (int h = 0; h < LN::HW; ++h)
            for (int k = 0; k < 6; ++k) {
                const double r = red[(c * LN::HW + h) * 6 + k];
                m[k] = (k == 5) ? fmax(m[k], r) : m[k] + r;
            }
        for (int k = 0; k < 5; ++k) {  // lambda = (C C^T)^{-1} C Qt
            double s = 0.0;
            for (int q = 0; q < 5; ++q) s = fma(pc.ginv[k * 5 + q], m[q], s);
            lam[c * 8 + k] = s;
        }
        if (maximag && cl < ncells) maximag[cl] = m[5];
    }
    __syncthreads();
    const double l0 = lam[sub * 8 + 0], l1 = lam[sub * 8 + 1], l2 = lam[sub * 8 + 2], l3 = lam[sub * 8 + 3],
                 l4 = lam[sub * 8 + 4];
    bool bad = false;
    if constexpr (!FWD) {
        // out = base + coef * (Qt - w C^T lambda) at nodes ln + k N^2: i1 = k, (i2, i3) = (a, b)
        const double cl23 = l0 + fv2 * l2 + fv3 * l3 + (fv2 * fv2 + fv3 * fv3) * l4;
        if (live) {
#pragma unroll
            for (int k = 0; k < N; ++k) {
                const double v1 = pc.dv * (k - N / 2);
                const double cl = fma(v1, fma(v1, l4, l1), cl23);
                const double q = sm[LN::at(k, a, b)].x - axis_coeff(N, k) * fw23 * cl;
                double v = coef * q;
                if (base) v += bv[k];
                bad |= !isfinite(v);
                out[(size_t)cell * N3 + (size_t)k * NN + ln] = v;
            }
        }
        if (bad) atomicOr(flag, 2);
    } else {
        // f* = base + coef * P_N(Qt) on the line (a, b, :), times s_m c_m, and its
        // forward transform: pass 1 in registers, pass 2 in smem, pass 3 to A_next
        const double v1 = pc.dv * (a - N / 2), v2 = pc.dv * (b - N / 2);
        const double cl12 = l0 + v1 * l1 + v2 * l2 + (v1 * v1 + v2 * v2) * l4;
        const double w12 = axis_coeff(N, a) * axis_coeff(N, b);
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const double v3 = pc.dv * (j - N / 2);
            const double cl = fma(v3, fma(v3, l4, l3), cl12);
            const double q = sm[LN::at(a, b, j)].x - w12 * axis_coeff(N, j) * dv3 * cl;
            double v = 0.0;
            if (live) {
                v = coef * q;
                if (base) v += bv[j];
                bad |= !isfinite(v);
            }
            double w = w12 * axis_coeff(N, j);
            if ((a + b + j) & 1) w = -w;
            x[j] = make_double2(v * w, 0.0);
        }
        if (bad) atomicOr(flag, 2);
        RegFFT<N, -1, N>::run(x);
        // the thread's own line: no other thread reads it after the barrier above
#pragma unroll
        for (int j = 0; j < N; ++j) sm[LN::at(a, b, j)] = x[j];
        __syncthreads();
        line_pass_axis1<N, -1>(sm, a, b);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < N; ++j) x[j] = sm[LN::at(j, a, b)];
        RegFFT<N, -1, N>::run(x);
        if constexpr (BOLTZ_LINE_TMA) {  // through a staging image over the cubes, as k_fwd_line_tma
            __syncthreads();
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const double s = ((j + a + b) & 1) ? -fwd_scale : fwd_scale;
                smem_line[(j * NN + ln) * CPB + sub] = make_double2(x[j].x * s, x[j].y * s);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (t == 0) {
                const long long cell0 = (long long)blockIdx.x * CPB;
                const int c0 = (int)(cell0 % kLanes) * 2, row0 = (int)(cell0 / kLanes) * N3;
#pragma unroll 1
                for (int j = 0; j < N; ++j) tma_store_2d(&tmNext, smem_line + j * NN * CPB, c0, row0 + j * NN);
                bulk_commit();
                bulk_wait_all();
            }
        } else {
#pragma unroll
            for (int j = 0; j < N; ++j) {
                const double s = ((j + a + b) & 1) ? -fwd_scale : fwd_scale;
                A_next[((size_t)g * N3 + (size_t)(j * N + a) * N + b) * kLanes + lane] =
                    make_double2(x[j].x * s, x[j].y * s);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// K3 with every HBM access by TMA (BOLTZ_LINE_INV2, N = 8, 16 with 16-byte
// aligned user arrays).  The passes run i1, i2, i3 -- the reverse of
// k_inv_line -- so that pass 1 reads the group rows plane by plane (one TMA box
// per i1 plane, landed on the cubes) and pass 3 leaves each thread the line
// (i1, i2, :) that the projection, the RK2 axpy, the user-layout base / out
// (swizzled line images, one TMA box per cell) and the fused forward
// transform's first pass all want.  Moments: per thread over i3, then the same
// fixed-order reduction as k_inv_line.
// ---------------------------------------------------------------------------
#ifndef BOLTZ_LINE_INV2
#define BOLTZ_LINE_INV2 1
#endif
template <int N, int CPB>
struct LineInv {
    static constexpr int F_BYTES = CPB * N * N * N * 8;  // base image / out staging (swizzled lines)
    static constexpr int SMEM = Line<N, CPB>::SMEM + F_BYTES + 1024 + 16;
};

template <int N, bool FWD, int CPB>
__global__ void __launch_bounds__(Line<N, CPB>::THREADS, Line<N, CPB>::MINB)
k_inv_line2(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmBase,
            const __grid_constant__ CUtensorMap tmOut, const __grid_constant__ CUtensorMap tmNext, int has_base,
            double* __restrict__ maximag, long long ncells, double scale, double coef, ProjConst pc,
            int* __restrict__ flag, double fwd_scale) {
    using LN = Line<N, CPB>;
    constexpr int N3 = LN::N3, NN = N * N;
    constexpr unsigned F_BYTES = LineInv<N, CPB>::F_BYTES;
    static_assert(N3 * CPB <= CPB * LN::CELL, "the group image fits over the cubes");
    extern __shared__ __align__(128) double2 smem_line_tma[];
    double2* cubes = smem_line_tma;
    double* red = reinterpret_cast<double*>(cubes + CPB * LN::CELL);  // [CPB][HW][6]
    double* lam = red + CPB * LN::HW * 6;                            // [CPB][8]
    char* img = reinterpret_cast<char*>(lam + CPB * 8);
    img += (1024 - (smem_u32(img) & 1023)) & 1023;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(img + F_BYTES);
    const int t = threadIdx.x, sub = LN::sub(t), ln = LN::line(t), a = ln / N, b = ln % N;
    double2* sm = cubes + sub * LN::CELL;
    const long long cell0 = (long long)blockIdx.x * CPB, cell = cell0 + sub;
    const bool live = cell < ncells;
    const int c0 = (int)(cell0 % kLanes) * 2, row0 = (int)(cell0 / kLanes) * N3;
    char* myline = img + sub * N3 * 8;  // this cell's line image; the thread's line is row ln
    if constexpr (BOLTZ_LINE_SPREAD) {
        // the barrier (expecting every byte) first, then each warp's elected lane
        // issues its share of the plane loads
        constexpr int W = LN::WARPS;
        if (t == 0) {
            mbar_init(bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            mbar_expect_tx(bar, (unsigned)(N3 * CPB * 16) + (has_base ? F_BYTES : 0u));
        }
        __syncthreads();
        const int w = t >> 5;
#pragma unroll
        for (int j = w; j < N; j += W) tma_load_2d_elect(cubes + j * NN * CPB, &tmB, c0, row0 + j * NN, bar);
        if (has_base && w == W - 1)
#pragma unroll
            for (int c = 0; c < CPB; ++c) tma_load_2d_elect(img + c * N3 * 8, &tmBase, 0, (int)((cell0 + c) * NN), bar);
    } else {
        if (t == 0) {
            mbar_init(bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            mbar_expect_tx(bar, (unsigned)(N3 * CPB * 16) + (has_base ? F_BYTES : 0u));
#pragma unroll 1
            for (int j = 0; j < N; ++j) tma_load_2d(cubes + j * NN * CPB, &tmB, c0, row0 + j * NN, bar);
            if (has_base)
#pragma unroll 1
                for (int c = 0; c < CPB; ++c) tma_load_2d(img + c * N3 * 8, &tmBase, 0, (int)((cell0 + c) * NN), bar);
        }
        __syncthreads();
    }
    mbar_wait(bar, 0);
    // pass 1 (axis 0, i1) from the group image: thread ln = (i2, i3)
    double2 x[N];
#pragma unroll
    for (int j = 0; j < N; ++j) x[j] = cubes[(j * NN + ln) * CPB + sub];
    double bv[N];  // the RK2 base on the thread's pass-3 line (i1, i2) = (a, b)
#pragma unroll
    for (int j = 0; j < N / 2; ++j) {
        const double2 u = has_base ? *reinterpret_cast<const double2*>(myline + swz<N>(ln * N * 8 + j * 16))
                                   : make_double2(0.0, 0.0);
        bv[2 * j] = u.x;
        bv[2 * j + 1] = u.y;
    }
    __syncthreads();  // the group image is consumed: the cubes take its place
    RegFFT<N, +1, N>::run(x);
#pragma unroll
    for (int j = 0; j < N; ++j) sm[LN::at(j, a, b)] = x[j];
    __syncthreads();
    line_pass_axis1<N, +1>(sm, a, b);
    __syncthreads();
    // pass 3 (axis 2, i3) in registers: Qt = Re(scale * par * s_k * z) on the line
    // (i1, i2) = (a, b), its moments over i3 and max|Im|
#pragma unroll
    for (int j = 0; j < N; ++j) x[j] = sm[LN::at(a, b, j)];
    RegFFT<N, +1, N>::run(x);
    const double dv3 = pc.dv * pc.dv * pc.dv;
    const double v1 = pc.dv * (a - N / 2), v2 = pc.dv * (b - N / 2);
    const double w12 = axis_coeff(N, a) * axis_coeff(N, b);
    const double fw12 = w12 * dv3;
    const double sg12 = ((a + b) & 1) ? -scale : scale;
    double s0 = 0.0, s3 = 0.0, s4 = 0.0, mi = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const double q = x[j].x * ((j & 1) ? -sg12 : sg12);
        x[j].x = q;
        const double v3 = pc.dv * (j - N / 2);
        const double cq = axis_coeff(N, j) * q;
        s0 += cq;
        s3 = fma(v3, cq, s3);
        s4 = fma(v3 * v3, cq, s4);
        mi = fmax(mi, fabs(x[j].y));
    }
    double part[6];
    part[0] = fw12 * s0;
    part[1] = v1 * part[0];
    part[2] = v2 * part[0];
    part[3] = fw12 * s3;
    part[4] = fw12 * fma(v1 * v1 + v2 * v2, s0, s4);
    part[5] = mi * fabs(scale);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        double v = part[k];
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            const double u = __shfl_xor_sync(0xffffffffu, v, o);
            v = (k == 5) ? fmax(v, u) : v + u;
        }
        if ((ln & 15) == 0) red[(sub * LN::HW + (ln >> 4)) * 6 + k] = v;
    }
    __syncthreads();
    if (t < CPB) {
        const int c = t;
        const long long cl = cell0 + c;
        double m[6] = {0, 0, 0, 0, 0, 0};
        for (int h = 0; h < LN::HW; ++h)
            for (int k = 0; k < 6; ++k) {
                const double r = red[(c * LN::HW + h) * 6 + k];
                m[k] = (k == 5) ? fmax(m[k], r) : m[k] + r;
            }
        for (int k = 0; k < 5; ++k) {  // lambda = (C C^T)^{-1} C Qt
            double s = 0.0;
            for (int q = 0; q < 5; ++q) s = fma(pc.ginv[k * 5 + q], m[q], s);
            lam[c * 8 + k] = s;
        }
        if (maximag && cl < ncells) maximag[cl] = m[5];
    }
    __syncthreads();
    const double l0 = lam[sub * 8 + 0], l1 = lam[sub * 8 + 1], l2 = lam[sub * 8 + 2], l3 = lam[sub * 8 + 3],
                 l4 = lam[sub * 8 + 4];
    // out / f* = base + coef * (Qt - w C^T lambda) on the line
    const double cl12 = l0 + v1 * l1 + v2 * l2 + (v1 * v1 + v2 * v2) * l4;
    bool bad = false;
    double v[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        const double v3 = pc.dv * (j - N / 2);
        const double cl = fma(v3, fma(v3, l4, l3), cl12);
        const double q = x[j].x - w12 * axis_coeff(N, j) * dv3 * cl;
        double r = 0.0;
        if (live) {
            r = coef * q;
            if (has_base) r += bv[j];
            bad |= !isfinite(r);
        }
        v[j] = r;
    }
    if (bad) atomicOr(flag, 2);
    if constexpr (!FWD) {
        // the line into its place in the image (only this thread touched it), then one box per cell
#pragma unroll
        for (int j = 0; j < N / 2; ++j)
            *reinterpret_cast<double2*>(myline + swz<N>(ln * N * 8 + j * 16)) = make_double2(v[2 * j], v[2 * j + 1]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (BOLTZ_LINE_SPREAD && t < 32) {  // warp 0, predicate inside the asm
#pragma unroll
            for (int c = 0; c < CPB; ++c) tma_store_2d_elect(&tmOut, img + c * N3 * 8, 0, (int)((cell0 + c) * NN));
            bulk_commit_wait_all_elect();
        } else if (!BOLTZ_LINE_SPREAD && t == 0) {
#pragma unroll 1
            for (int c = 0; c < CPB; ++c) tma_store_2d(&tmOut, img + c * N3 * 8, 0, (int)((cell0 + c) * NN));
            bulk_commit();
            bulk_wait_all();
        }
    } else {
        // f* times s_m c_m and its forward transform: pass 1 in registers, pass 2
        // in smem, pass 3 to the staging image, stored by TMA into A_next
#pragma unroll
        for (int j = 0; j < N; ++j) {
            double w = w12 * axis_coeff(N, j);
            if ((a + b + j) & 1) w = -w;
            x[j] = make_double2(v[j] * w, 0.0);
        }
        RegFFT<N, -1, N>::run(x);
        // the thread's own line: no other thread reads it after the barrier above
#pragma unroll
        for (int j = 0; j < N; ++j) sm[LN::at(a, b, j)] = x[j];
        __syncthreads();
        line_pass_axis1<N, -1>(sm, a, b);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < N; ++j) x[j] = sm[LN::at(j, a, b)];
        RegFFT<N, -1, N>::run(x);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const double s = ((j + a + b) & 1) ? -fwd_scale : fwd_scale;
            cubes[(j * NN + ln) * CPB + sub] = make_double2(x[j].x * s, x[j].y * s);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if constexpr (BOLTZ_LINE_SPREAD) {  // each warp's elected lane stores its planes
            const int w = t >> 5;
#pragma unroll
            for (int j = w; j < N; j += LN::WARPS) tma_store_2d_elect(&tmNext, cubes + j * NN * CPB, c0, row0 + j * NN);
            bulk_commit_wait_all_elect();
        } else if (t == 0) {
#pragma unroll 1
            for (int j = 0; j < N; ++j) tma_store_2d(&tmNext, cubes + j * NN * CPB, c0, row0 + j * NN);
            bulk_commit();
            bulk_wait_all();
        }
    }
}

}  // namespace boltz_gpu
