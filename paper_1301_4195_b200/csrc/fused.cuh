// fused.cuh -- single-kernel K1 and K3 for grids whose N^3 cube fits in shared
// memory (N <= 24): one CTA owns CPB whole cells, does all three FFT axes in
// shared memory, and touches HBM exactly once per operand.
//
//   k_fwd_fused:     user f [cell][N^3]  -> group fhat (forward, fourier.hpp:11-12)
//   k_inv_project:   group s_k*Qhat       -> out = base + coef * P_N(Re iFFT)  (+ max|Im|)
//                    (inverse fourier.hpp:15-17, projection SPEC.md:204-212,
//                     RK2 axpy SPEC.md:383-391)
//
// HBM traffic per cell (N=16): forward 32 KiB in + 64 KiB out; inverse+project
// 64 KiB in + 32 KiB base + 32 KiB out -- versus 3 read+write sweeps each for
// the multi-pass path (transforms.cuh), which remains for N = 32.
//
// Shared layout per cell: [i1][i2][i3] complex with rows padded to N+1 so the
// three axis passes are bank-conflict free for 16 B accesses.
#pragma once
#include "common.cuh"
#include "fft.cuh"

namespace boltz_gpu {

template <int N>
struct Fused {
    static constexpr int N3 = N * N * N;
    // Shared layout per cell: [i1][i2][i3] complex.  Rows are padded to N+1 when
    // that fits (N <= 16), which makes the three axis passes conflict-free for
    // 16 B accesses; otherwise (N = 24: 221 KB unpadded) i3 is XOR-swizzled with
    // the low 3 bits of i2 -- the same effect without the padding.
    static constexpr bool PAD = N * N * (N + 1) * 16 <= 200 * 1024;
    static constexpr int ROW = PAD ? N + 1 : N;       // row length (complex elements)
    static constexpr int CELL = N * N * ROW;          // complex elements per cell in smem
    static constexpr int CELL_BYTES = CELL * 16;
    // cells per block: largest power of two <= 32 whose cubes fit in ~200 KB
#ifndef BOLTZ_FUSED_BUDGET_KB
#define BOLTZ_FUSED_BUDGET_KB 200
#endif
    static constexpr int BUDGET = BOLTZ_FUSED_BUDGET_KB * 1024;
    static constexpr int CPB = (CELL_BYTES * 32 <= BUDGET)   ? 32
                               : (CELL_BYTES * 16 <= BUDGET) ? 16
                               : (CELL_BYTES * 8 <= BUDGET)  ? 8
                               : (CELL_BYTES * 4 <= BUDGET)  ? 4
                               : (CELL_BYTES * 2 <= BUDGET)  ? 2
                                                             : 1;
#ifndef BOLTZ_FUSED_THREADS
#define BOLTZ_FUSED_THREADS 512
#endif
    // the N=24 register FFT needs ~130 registers: 256 threads
    static constexpr int THREADS = N > 16 ? 256 : BOLTZ_FUSED_THREADS;
    static constexpr int RED_BYTES = (THREADS / 32) * CPB * 6 * 8;
    static constexpr int SMEM_MAX = 232448;  // 227 KB opt-in dynamic shared memory per block
    // real staging (CPB x N^3 doubles): the forward's f, the inverse's RK2 base,
    // both fetched by cp.async so every load of the tile is in flight at once
    // (only where it fits beside the cubes: not at N = 24)
    static constexpr int STAGE_BYTES =
        CPB * CELL_BYTES + RED_BYTES + CPB * N3 * 8 <= SMEM_MAX ? CPB * N3 * 8 : 0;
    static constexpr int SMEM = CPB * CELL_BYTES + RED_BYTES + STAGE_BYTES;  // cubes + reduction scratch + staging
    static constexpr bool FITS = CPB * CELL_BYTES + RED_BYTES <= SMEM_MAX;
    __device__ static int at(int i1, int i2, int i3) {
        return PAD ? (i1 * N + i2) * ROW + i3 : (i1 * N + i2) * N + (i3 ^ (i2 & 7));
    }
};

// in-place FFT of every line along AXIS of the CPB cubes in shared memory
template <int N, int AXIS, int SIGN>
__device__ __forceinline__ void smem_axis_pass(double2* sm) {
    using F = Fused<N>;
    for (int r = threadIdx.x; r < F::CPB * N * N; r += F::THREADS) {
        const int c = r / (N * N), q = r % (N * N), a = q / N, b = q % N;
        double2* base = sm + c * F::CELL;
        auto pos = [&](int j) {
            return AXIS == 2 ? F::at(a, b, j) : AXIS == 1 ? F::at(a, j, b) : F::at(j, a, b);
        };
        double2 x[N];
#pragma unroll
        for (int j = 0; j < N; ++j) x[j] = base[pos(j)];
        RegFFT<N, SIGN, N>::run(x);
#pragma unroll
        for (int j = 0; j < N; ++j) base[pos(j)] = x[j];
    }
}

// CPB consecutive user-layout cells [cell0, cell0 + CPB) of src -> stage
// (CPB x N^3 doubles) with 16-byte cp.async (one commit group); cells past
// ncells are zero.  src must be 16-byte aligned (the callers check).
template <int N>
__device__ __forceinline__ void stage_cells(double* stage, const double* __restrict__ src, long long cell0,
                                            long long ncells) {
    using F = Fused<N>;
    constexpr int N3 = F::N3, CH = N3 / 2;  // 16-byte chunks per cell
    for (int t = threadIdx.x; t < F::CPB * CH; t += F::THREADS) {
        const int c = t / CH, j = t % CH;
        double* d = stage + (size_t)c * N3 + 2 * j;
        if (cell0 + c < ncells) cp_async16(d, src + (size_t)(cell0 + c) * N3 + 2 * j);
        else d[0] = d[1] = 0.0;
    }
    cp_async_commit();
}

// group-layout complex cube of CPB cells -> padded smem cubes (one commit group)
template <int N>
__device__ __forceinline__ void stage_group(double2* sm, const double2* __restrict__ B, long long g, int lane0) {
    using F = Fused<N>;
    constexpr int N3 = F::N3;
    for (int t = threadIdx.x; t < F::CPB * N3; t += F::THREADS) {
        const int idx = t / F::CPB, c = t % F::CPB;
        const int i1 = idx / (N * N), i2 = (idx / N) % N, i3 = idx % N;
        cp_async16(sm + c * F::CELL + F::at(i1, i2, i3), B + ((size_t)g * N3 + idx) * kLanes + lane0 + c);
    }
    cp_async_commit();
}

// grid = ngroups * 32 / CPB blocks; block b covers cells [b*CPB, b*CPB+CPB)
template <int N>
__global__ void __launch_bounds__(Fused<N>::THREADS)
k_fwd_fused(const double* __restrict__ f, double2* __restrict__ A, long long ncells, double scale,
            int* __restrict__ flag) {
    using F = Fused<N>;
    constexpr int N3 = F::N3;
    extern __shared__ __align__(16) double2 sm[];
    double* stage = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + F::CPB * F::CELL_BYTES + F::RED_BYTES);
    const long long cell0 = (long long)blockIdx.x * F::CPB;
    const bool staged = F::STAGE_BYTES > 0 && (reinterpret_cast<uintptr_t>(f) & 15) == 0;
    if (staged) {
        stage_cells<N>(stage, f, cell0, ncells);
        cp_async_wait_all();
        __syncthreads();
    }
    bool bad = false;
    // pre-multiply by s_m c_m (coalesced per cell)
#pragma unroll 4
    for (int t = threadIdx.x; t < F::CPB * N3; t += F::THREADS) {
        const int c = t / N3, idx = t % N3;
        const long long cell = cell0 + c;
        const int i1 = idx / (N * N), i2 = (idx / N) % N, i3 = idx % N;
        double v = staged ? stage[t] : (cell < ncells ? f[(size_t)cell * N3 + idx] : 0.0);
        bad |= !isfinite(v);
        double w = axis_coeff(N, i1) * axis_coeff(N, i2) * axis_coeff(N, i3);
        if ((i1 + i2 + i3) & 1) w = -w;
        sm[c * F::CELL + F::at(i1, i2, i3)] = make_double2(v * w, 0.0);
    }
    if (bad) atomicOr(flag, 1);
    __syncthreads();
    smem_axis_pass<N, 2, -1>(sm);
    __syncthreads();
    smem_axis_pass<N, 1, -1>(sm);
    __syncthreads();
    smem_axis_pass<N, 0, -1>(sm);
    __syncthreads();
    // post-multiply scale*par*s_k and scatter into the group layout:
    // CPB consecutive lanes of one group -> CPB*16 contiguous bytes per node
    const long long g = cell0 / kLanes;
    const int lane0 = (int)(cell0 % kLanes);
#pragma unroll 4
    for (int t = threadIdx.x; t < F::CPB * N3; t += F::THREADS) {
        const int idx = t / F::CPB, c = t % F::CPB;
        const int i1 = idx / (N * N), i2 = (idx / N) % N, i3 = idx % N;
        const double s = ((i1 + i2 + i3) & 1) ? -scale : scale;
        const double2 z = sm[c * F::CELL + F::at(i1, i2, i3)];
        A[((size_t)g * N3 + idx) * kLanes + lane0 + c] = make_double2(z.x * s, z.y * s);
    }
}

// FWD = true fuses the next RK2 stage's forward transform: instead of writing
// out = base + coef*Q, the kernel transforms that value in shared memory and
// writes its fhat (times fwd_scale) into the group layout A_next.
template <int N, bool FWD = false>
__global__ void __launch_bounds__(Fused<N>::THREADS)
k_inv_project(const double2* __restrict__ B, const double* __restrict__ base, double* __restrict__ out,
              double* __restrict__ maximag, long long ncells, double scale, double coef, ProjConst pc,
              int* __restrict__ flag, double2* __restrict__ A_next = nullptr, double fwd_scale = 0.0) {
    using F = Fused<N>;
    constexpr int N3 = F::N3;
    constexpr int CPB = F::CPB;
    extern __shared__ __align__(16) double2 sm[];
    double* red = reinterpret_cast<double*>(sm + CPB * F::CELL);  // [warps][CPB][6], after the cubes
    double* stage = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + CPB * F::CELL_BYTES + F::RED_BYTES);
    __shared__ double lam[CPB][5];
    const long long cell0 = (long long)blockIdx.x * CPB;
    const long long g = cell0 / kLanes;
    const int lane0 = (int)(cell0 % kLanes);
    // every load of the tile in flight at once: the cube, then the RK2 base
    // (which is only needed after the transform and the projection)
    stage_group<N>(sm, B, g, lane0);
    const bool staged = F::STAGE_BYTES > 0 && base && (reinterpret_cast<uintptr_t>(base) & 15) == 0;
    if (staged) {
        stage_cells<N>(stage, base, cell0, ncells);
        cp_async_wait_1();
    } else {
        cp_async_wait_all();
    }
    __syncthreads();
    smem_axis_pass<N, 2, +1>(sm);
    __syncthreads();
    smem_axis_pass<N, 1, +1>(sm);
    __syncthreads();
    smem_axis_pass<N, 0, +1>(sm);
    __syncthreads();
    // Qt = Re(scale*par*s_k*z) in place (.x); moments + max|Im| per cell with a
    // deterministic reduction (fixed strided partials, shuffle tree, warps in order)
    const double dv3 = pc.dv * pc.dv * pc.dv;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // THREADS a multiple of N^2: every node a thread visits has the same (i2, i3),
    // so the per-node weights and moments factor into per-thread constants and
    // three FMAs per node (sums over i1 only; the result is reassembled below)
    constexpr bool kFixed23 = F::THREADS % (N * N) == 0;
    const int f2 = (threadIdx.x / N) % N, f3 = threadIdx.x % N;
    const double fv2 = pc.dv * (f2 - N / 2), fv3 = pc.dv * (f3 - N / 2);
    const double fw23 = axis_coeff(N, f2) * axis_coeff(N, f3) * dv3;
    for (int c = 0; c < CPB; ++c) {
        double part[6] = {0, 0, 0, 0, 0, 0};
        if constexpr (kFixed23) {
            double s0 = 0.0, s1 = 0.0, s4 = 0.0, mi = 0.0;
            const double sg23 = ((f2 + f3) & 1) ? -scale : scale;
            for (int idx = threadIdx.x; idx < N3; idx += F::THREADS) {
                const int i1 = idx / (N * N);
                double2* p = sm + c * F::CELL + F::at(i1, f2, f3);
                const double2 z = *p;
                const double q = z.x * ((i1 & 1) ? -sg23 : sg23);
                p->x = q;
                const double v1 = pc.dv * (i1 - N / 2);
                const double cq = axis_coeff(N, i1) * q;
                s0 += cq;
                s1 = fma(v1, cq, s1);
                s4 = fma(v1 * v1, cq, s4);
                mi = fmax(mi, fabs(z.y));
            }
            part[0] = fw23 * s0;
            part[1] = fw23 * s1;
            part[2] = fv2 * part[0];
            part[3] = fv3 * part[0];
            part[4] = fw23 * fma(fv2 * fv2 + fv3 * fv3, s0, s4);
            part[5] = mi * fabs(scale);
        } else {
            for (int idx = threadIdx.x; idx < N3; idx += F::THREADS) {
                const int i1 = idx / (N * N), i2 = (idx / N) % N, i3 = idx % N;
                double2* p = sm + c * F::CELL + F::at(i1, i2, i3);
                const double2 z = *p;
                const double s = ((i1 + i2 + i3) & 1) ? -scale : scale;
                const double q = z.x * s;
                p->x = q;
                const double v1 = pc.dv * (i1 - N / 2), v2 = pc.dv * (i2 - N / 2), v3 = pc.dv * (i3 - N / 2);
                const double wq = axis_coeff(N, i1) * axis_coeff(N, i2) * axis_coeff(N, i3) * dv3 * q;
                part[0] += wq;
                part[1] += v1 * wq;
                part[2] += v2 * wq;
                part[3] += v3 * wq;
                part[4] += (v1 * v1 + v2 * v2 + v3 * v3) * wq;
                part[5] = fmax(part[5], fabs(z.y * scale));
            }
        }
#pragma unroll
        for (int a = 0; a < 6; ++a) {
            double v = part[a];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double u = __shfl_xor_sync(0xffffffffu, v, o);
                v = (a == 5) ? fmax(v, u) : v + u;
            }
            if (lane == 0) red[(wid * CPB + c) * 6 + a] = v;
        }
    }
    __syncthreads();
    if (threadIdx.x < CPB) {
        const int c = threadIdx.x;
        double m[6] = {0, 0, 0, 0, 0, 0};
        for (int w = 0; w < F::THREADS / 32; ++w)
            for (int a = 0; a < 6; ++a) {
                const double r = red[(w * CPB + c) * 6 + a];
                m[a] = (a == 5) ? fmax(m[a], r) : m[a] + r;
            }
        for (int a = 0; a < 5; ++a) {
            double t = 0.0;
            for (int b = 0; b < 5; ++b) t = fma(pc.ginv[a * 5 + b], m[b], t);
            lam[c][a] = t;
        }
        if (maximag && cell0 + c < ncells) maximag[cell0 + c] = m[5];
    }
    __syncthreads();
    if (staged) {
        cp_async_wait_all();
        __syncthreads();
    }
    bool bad = false;
#pragma unroll 4
    for (int t = threadIdx.x; t < CPB * N3; t += F::THREADS) {
        const int c = t / N3, idx = t % N3;
        const long long cell = cell0 + c;
        if (!FWD && cell >= ncells) continue;
        const double bv = staged ? stage[t] : (base && cell < ncells ? base[(size_t)cell * N3 + idx] : 0.0);
        const int i1 = idx / (N * N), i2 = kFixed23 ? f2 : (idx / N) % N, i3 = kFixed23 ? f3 : idx % N;
        const double v1 = pc.dv * (i1 - N / 2);
        double wq, cl;
        if constexpr (kFixed23) {
            wq = axis_coeff(N, i1) * fw23;
            cl = fma(v1, fma(v1, lam[c][4], lam[c][1]),
                     lam[c][0] + fv2 * lam[c][2] + fv3 * lam[c][3] + (fv2 * fv2 + fv3 * fv3) * lam[c][4]);
        } else {
            const double v2 = pc.dv * (i2 - N / 2), v3 = pc.dv * (i3 - N / 2);
            wq = axis_coeff(N, i1) * axis_coeff(N, i2) * axis_coeff(N, i3) * dv3;
            cl = lam[c][0] + v1 * lam[c][1] + v2 * lam[c][2] + v3 * lam[c][3] + (v1 * v1 + v2 * v2 + v3 * v3) * lam[c][4];
        }
        double2* p = sm + c * F::CELL + F::at(i1, i2, i3);
        const double q = p->x - wq * cl;
        const size_t o = (size_t)cell * N3 + idx;
        if constexpr (FWD) {
            // the RK2 stage value f* = base + coef*Q never leaves the SM: it is
            // pre-multiplied by s_m c_m for the forward transform in place
            double v = 0.0;
            if (cell < ncells) {
                v = coef * q;
                if (base) v += bv;
                bad |= !isfinite(v);
            }
            double w = axis_coeff(N, i1) * axis_coeff(N, i2) * axis_coeff(N, i3);
            if ((i1 + i2 + i3) & 1) w = -w;
            *p = make_double2(v * w, 0.0);
        } else {
            double v = coef * q;
            if (base) v += bv;
            bad |= !isfinite(v);
            out[o] = v;
        }
    }
    if (bad) atomicOr(flag, 2);
    if constexpr (FWD) {
        __syncthreads();
        smem_axis_pass<N, 2, -1>(sm);
        __syncthreads();
        smem_axis_pass<N, 1, -1>(sm);
        __syncthreads();
        smem_axis_pass<N, 0, -1>(sm);
        __syncthreads();
#pragma unroll 4
        for (int t = threadIdx.x; t < CPB * N3; t += F::THREADS) {
            const int idx = t / CPB, c = t % CPB;
            const int i1 = idx / (N * N), i2 = (idx / N) % N, i3 = idx % N;
            const double s = ((i1 + i2 + i3) & 1) ? -fwd_scale : fwd_scale;
            const double2 z = sm[c * F::CELL + F::at(i1, i2, i3)];
            A_next[((size_t)g * N3 + idx) * kLanes + lane0 + c] = make_double2(z.x * s, z.y * s);
        }
    }
}

}  // namespace boltz_gpu
