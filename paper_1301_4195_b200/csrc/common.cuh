// common.cuh -- shared constants and helpers for the boltz sm_100a kernels.
//
// Device data layout ("group layout"): the cells of a batch
// are grouped 32 at a time; a group stores every velocity/Fourier node of its
// 32 cells contiguously, cell fastest:
//     X[g][idx][lane]        idx = (i1*N + i2)*N + i3   (velocity_grid.hpp:30-32)
// so a warp whose lane == cell reads one node of 32 cells as one coalesced
// 512 B (complex) / 256 B (real) transaction.  All per-cell arithmetic of the
// collision path is then warp-uniform in control flow and in the weight-table
// address, which is what lets Ĝ be read once per warp for 32 cells.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace boltz_gpu {

constexpr int kLanes = 32;          // cells per group
constexpr double kPi = 3.14159265358979323846264338327950288;

// Supported velocity-grid sizes (template instantiations).  SPEC.md:41 allows
// any even N >= 4; the library instantiates the ones the configs and tests use.
#define BOLTZ_FOR_EACH_N(X) X(4) X(6) X(8) X(12) X(16) X(24) X(32)

// Twiddle tables, one per supported N, concatenated in constant memory:
// c_tw[tw_offset(N) + j] = exp(-2*pi*i*j/N), j in [0, N).
__host__ __device__ constexpr int tw_offset(int n) {
    return n == 4 ? 0 : n == 6 ? 4 : n == 8 ? 10 : n == 12 ? 18 : n == 16 ? 30 : n == 24 ? 46 : n == 32 ? 70 : -1;
}
constexpr int kTwTotal = 102;

// (CC^T)^{-1} and the grid scalars used by the projection epilogue, set per
// context before each launch sequence (cheap: 40 doubles).
struct ProjConst {
    double ginv[25];   // (C C^T)^{-1}, row-major 5x5
    double dv;         // velocity mesh size
    double half;       // N/2 as double
};

__device__ __forceinline__ double2 ldg2(const double2* p) { return __ldg(p); }

__host__ __device__ __forceinline__ double axis_coeff(int n, int k) { return (k == 0 || k == n - 1) ? 0.5 : 1.0; }

// cp.async (LDGSTS) 16-byte global -> shared copies and their group fences
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

}  // namespace boltz_gpu
