// gen.cuh -- on-device generation of the folded table H:
// evaluates Ĝ at every (k, m) and (k, σm) the convolution consumes directly
// from the closed forms / quadrature of weight_math.h (the same code the host
// generator runs), so a context can be built without the dense N^6 host table
// (8.6 GB at N=32).  Folding as in k_build_H (conv.cuh).
#pragma once
#include "common.cuh"
#include "weight_math.h"

namespace boltz_gpu {

struct GenParams {
    double lambda, beta, r0, dz2, w3;
    int panels, n;
    boltz_w::Gauss16 gl;
};

__global__ void k_gen_H(double* __restrict__ H, const int4* __restrict__ entk, const short2* __restrict__ term,
                        int nent, int slab, GenParams gp) {
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= (long long)nent * slab) return;
    const int e = (int)(tid / slab), pos = (int)(tid % slab);
    const int4 q = entk[e];
    const short2 km = term[pos];
    double out = 0.0;
    if (km.x >= 0) {
        const int n = gp.n, h = n / 2;
        const int k1 = q.x, k2 = q.y, m1 = q.z, m2 = q.w, k3 = km.x, m3 = km.y;
        const int s1 = k1 - m1 + h, s2 = k2 - m2 + h, s3 = k3 - m3 + h;
        const double wm = axis_coeff(n, m1) * axis_coeff(n, m2) * axis_coeff(n, m3) * gp.w3;
        const double ws = axis_coeff(n, s1) * axis_coeff(n, s2) * axis_coeff(n, s3) * gp.w3;
        auto G = [&](int a1, int a2, int a3) {
            return boltz_w::lattice_weight(gp.lambda, gp.beta, gp.r0, gp.panels, gp.gl, gp.dz2, k1 - h, k2 - h,
                                           k3 - h, a1 - h, a2 - h, a3 - h);
        };
        const bool self_row = (m1 == s1) && (m2 == s2);
        if (!self_row || m3 < s3) out = G(m1, m2, m3) * wm + G(s1, s2, s3) * ws;
        else if (m3 == s3) out = G(m1, m2, m3) * wm;
    }
    H[(size_t)e * slab + pos] = out;
}

}  // namespace boltz_gpu
