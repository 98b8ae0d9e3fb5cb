// FP64 latency / per-warp throughput microbenchmark (development aid).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, long long* cyc, int iters, double a, double b) {
    double x[CH];
    for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-9 + i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) x[i] = fma(x[i], a, b);
    }
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < CH; ++i) s += x[i];
    if (s == 1234.5) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int CH>
void run(int warps) {
    double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8 * 1024);
    int iters = 4096;
    k<CH><<<1, 32 * warps>>>(o, c, iters, 0.999999, 1e-6);
    k<CH><<<1, 32 * warps>>>(o, c, iters, 0.999999, 1e-6);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("chains=%2d warps/CTA=%2d: %.2f cycles per DFMA per warp-chain-step; %.2f warp-DFMA/cycle/SM\n", CH, warps,
           (double)h / iters, (double)CH * iters * warps / h);
    cudaFree(o); cudaFree(c);
}
int main() {
    run<1>(1); run<2>(1); run<4>(1); run<8>(1); run<16>(1); run<8>(4); run<16>(4); run<8>(8); run<16>(8);
    return 0;
}
