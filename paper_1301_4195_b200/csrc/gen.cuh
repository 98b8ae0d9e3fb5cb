// gen.cuh -- on-device generation of the folded table H:
// evaluates Ĝ at every (k, m) and (k, σm) the convolution consumes directly
// from the closed forms / quadrature of weight_math.h (the same code the host
// generator runs), so a context can be built without the dense N^6 host table
// (8.6 GB at N=32).  Folding as in k_build_H (conv.cuh).
#pragma once
#include "common.cuh"
#include "conv.cuh"
#include "weight_math.h"

namespace boltz_gpu {

struct GenParams {
    double lambda, beta, r0, dz2, w3;
    int panels, n;
    boltz_w::Gauss16 gl;
};

// every entry e < nent (meta / TermSet as in k_build_H, conv.cuh)
__global__ void k_gen_H(double* __restrict__ H, const int4* __restrict__ entk, const int2* __restrict__ meta,
                        int nent, TermSet ts, GenParams gp) {
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= (long long)nent * ts.slab_max) return;
    const int e = (int)(tid / ts.slab_max), pos = (int)(tid % ts.slab_max);
    const int2 mt = meta[e];
    if (pos >= ts.slab[mt.y]) return;
    int4 q = entk[e];
    short2 km = ts.term[ts.off[mt.y] + pos];
    if (km.x >= kMirrorTermFlag) {  // a partner-row term (k_conv_mirror2)
        km.x -= kMirrorTermFlag;
        q = mirror_q(gp.n, q);
    }
    double out = 0.0;
    if (km.x >= 0) {
        const int h = gp.n / 2;
        out = folded_h(gp.n, gp.w3, q, km, [&](int k3, int a1, int a2, int a3) {
            return boltz_w::lattice_weight(gp.lambda, gp.beta, gp.r0, gp.panels, gp.gl, gp.dz2, q.x - h, q.y - h,
                                           k3 - h, a1 - h, a2 - h, a3 - h);
        });
    }
    H[(size_t)(unsigned)mt.x + pos] = out;
}

}  // namespace boltz_gpu
