// Upper bounds of the K2 inner loop (development aid).  N=16, T=16 band of
// k_conv_pipe; mode 0: operands in registers/smem, no row switch; mode 1: +y
// reload from smem every row; mode 2: + cp.async of the next row's x/y/H from
// global (L2-resident) and the wait/syncwarp at the row boundary.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1301_4195_b200/csrc/conv.cuh"
using namespace boltz_gpu;
constexpr int N = 16, T = 16;
template <int MODE>
__global__ void __launch_bounds__(128, 1) k(double* out, const double2* __restrict__ gsrc, int rows) {
    extern __shared__ __align__(16) char smem[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double2* wx = reinterpret_cast<double2*>(smem) + w * (3 * N * 32 + 2 * 96);  // x[2], y, H[2]
    for (int i = lane; i < 3 * N * 32 + 2 * 96; i += 32) wx[i] = make_double2(1e-3 * i, 2e-3 * i);
    __syncwarp();
    double2 acc[T], y[T];
#pragma unroll
    for (int i = 0; i < T; ++i) { acc[i] = make_double2(0, 0); y[i] = make_double2(lane * 1e-3 + i, i * 1e-3); }
    const double2* g = gsrc + (size_t)(blockIdx.x * 4 + w) * 4096;
    for (int r = 0; r < rows; ++r) {
        const int cur = r & 1;
        if (MODE >= 2) {
            __syncwarp();
            double2* xn = wx + (cur ^ 1) * N * 32;
            double2* yn = wx + 2 * N * 32;
            double2* hn = wx + 3 * N * 32 + (cur ^ 1) * 96;
            const double2* src = g + (r & 7) * 512;
#pragma unroll
            for (int j = 0; j < N; ++j) {
                cp_async16(xn + j * 32 + lane, src + j * 32 + lane);
                cp_async16(yn + j * 32 + lane, src + 256 + j * 32 + lane);
            }
            for (int o = lane; o < 96; o += 32) cp_async16(hn + o, src + o);
            cp_async_commit();
        }
        const double2* x = wx + cur * N * 32;
        const double2* h = wx + 3 * N * 32 + cur * 96;
        int p = 0;
        double2 hb = make_double2(0, 0);
        auto xat = [&](int m3) { return x[m3 * 32 + lane]; };
        band_tile<N, T, 1, 0, 0>(acc, y, xat, h, p, hb, [](int, int) {});
        if (MODE >= 2) { cp_async_wait_all(); __syncwarp(); }
        if (MODE >= 1) {
            const double2* ys = wx + 2 * N * 32;
#pragma unroll
            for (int j = 0; j < T; ++j) y[j] = ys[j * 32 + lane];
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < T; ++i) s += acc[i].x + acc[i].y;
    if (s == 1.2345) out[0] = s;
}
template <int MODE>
void run(int sms, double* o, const double2* g) {
    const int smem = 4 * (3 * N * 32 + 2 * 96) * 16;
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int ctas_per_sm : {2}) {
        int rows = 2000;
        k<MODE><<<sms * ctas_per_sm, 128, smem>>>(o, g, 10);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        k<MODE><<<sms * ctas_per_sm, 128, smem>>>(o, g, rows);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double terms = 192.0 * rows * 128 * sms * ctas_per_sm;
        printf("mode %d CTAs/SM=%d: %.2f TFLOP/s executed, err=%s\n", MODE, ctas_per_sm,
               terms * 12 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
}
int main() {
    double* o; cudaMalloc(&o, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double2* g; cudaMalloc(&g, ((size_t)sms * 2 * 4 + 2) * 4096 * 16); cudaMemset(g, 0, ((size_t)sms * 2 * 4 + 2) * 4096 * 16);
    run<0>(sms, o, g); run<1>(sms, o, g); run<2>(sms, o, g);
    return 0;
}
