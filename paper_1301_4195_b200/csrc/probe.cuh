// probe.cuh -- FP64 peak probe.  MEASURED_PEAKS.json has no FP64 entry, so
// bench.py measures the DFMA roofline denominator in-run: every SM runs 32
// warps of 8 independent DFMA chains (no memory traffic).
#pragma once
#include "common.cuh"

namespace boltz_gpu {

__global__ void __launch_bounds__(256) k_dfma_probe(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = 1e-9 * threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1234.5678) out[0] = s;  // never true; keeps the chains live
}

}  // namespace boltz_gpu
