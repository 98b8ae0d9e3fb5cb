// transport.cuh -- K4: second-order finite-volume transport on a non-uniform
// 1D grid and the physical-end ghost fill
// (linear extrapolation SPEC.md:318; diffuse Maxwell wall SPEC.md:333-341).
// Elementwise over (cell, velocity node); user layout field[cell][N^3] with
// two ghost cells per side, so consecutive threads touch
// consecutive nodes of one cell (coalesced).  HBM-bound: one load per f value
// (sliding stencil), per-cell geometry hoisted out of the node loop.
#pragma once
#include "common.cuh"

namespace boltz_gpu {

__device__ __forceinline__ double minmod3(double a, double b, double c) {
    if (a > 0 && b > 0 && c > 0) return fmin(a, fmin(b, c));
    if (a < 0 && b < 0 && c < 0) return fmax(a, fmax(b, c));
    return 0.0;
}

// Per-cell geometry of the 5-cell stencil around interior cell ce: inverse
// centre distances of the three minmod candidates of cells ce-1, ce, ce+1, their
// half widths, and dt/dx[ce].  Scalars per cell, so a block (one cell) computes
// them once instead of 9 FP64 divisions per velocity node.
struct StencilCoef {
    double r1[3], r2[3], r3[3];  // 1/(x[c+1]-x[c]), 1/(x[c]-x[c-1]), 1/(x[c+1]-x[c-1]), c = ce-1+d
    double hdx[3];               // 0.5 * dx[c]
};

__device__ __forceinline__ StencilCoef stencil_coef(long long ce, const double* __restrict__ x,
                                                    const double* __restrict__ dx) {
    StencilCoef k;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const long long c = ce - 1 + d;
        k.r1[d] = 1.0 / (x[c + 1] - x[c]);
        k.r2[d] = 1.0 / (x[c] - x[c - 1]);
        k.r3[d] = 1.0 / (x[c + 1] - x[c - 1]);
        k.hdx[d] = 0.5 * dx[c];
    }
    return k;
}

// Upwind fluxes through the left and right faces of interior cell ce at
// velocity node j: minmod slopes from the 5-cell stencil,
// each cell's own half-width, zero slope in the wall ghost / wall cell.
// Shared by the FV step and the boundary-flux ledger (bitwise the same faces).
template <int N>
__device__ __forceinline__ void face_fluxes(const double* __restrict__ f, long long ce, int j, long long ncl,
                                            const StencilCoef& k, int wl, int wr, double dv, double& fc, double& Fl,
                                            double& Fr) {
    constexpr int N3 = N * N * N;
    const double v1 = dv * (j / (N * N) - N / 2);
    double fv[5];
#pragma unroll
    for (int d = 0; d < 5; ++d) fv[d] = f[(ce - 2 + d) * N3 + j];
    double sg[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const long long c = ce - 1 + d;
        const double fm = fv[d], f0 = fv[d + 1], fp = fv[d + 2];
        double s = minmod3((fp - f0) * k.r1[d], (f0 - fm) * k.r2[d], (fp - fm) * k.r3[d]);
        if (wl && (c == 1 || c == 2)) s = 0.0;
        if (wr && (c == ncl + 2 || c == ncl + 1)) s = 0.0;
        sg[d] = s;
    }
    if (v1 >= 0.0) {
        Fl = v1 * (fv[1] + k.hdx[0] * sg[0]);
        Fr = v1 * (fv[2] + k.hdx[1] * sg[1]);
    } else {
        Fl = v1 * (fv[2] - k.hdx[1] * sg[1]);
        Fr = v1 * (fv[3] - k.hdx[2] * sg[2]);
    }
    fc = fv[2];
}

// grid = (ceil(N^3/512), ceil(ncl/kTrCells)): a thread owns velocity nodes
// 2p, 2p+1 (16-byte loads) of kTrCells consecutive interior cells and slides the 5-cell stencil along
// them, so each f value is loaded once (not 5 times), each minmod slope and
// each face flux is computed once and shared by its two cells -- the same
// arithmetic, face for face, as face_fluxes (bitwise).  Per-cell geometry
// (inverse distances, half widths, dt/dx) is computed once per block.
// Ghosts are copied through by the first / last chunk.
// out = alpha*base + (1-alpha)*(f - dt/dx (F_{j+1/2} - F_{j-1/2}))   (base may be null)
// -- the second stage of the SSP-RK2 transport sub-step fused in.
// Peer mode (peer != 0) fuses the halo exchange into the step: the two first
// and two last updated interior cells are also stored straight into the
// neighbours' output fields (left_dst: the left rank's ghosts ncl_L+2, ncl_L+3;
// right_dst: the right rank's ghosts 0, 1 -- peer memory over NVLink, or
// another field of the same device), and this rank's own ghost rows are NOT
// written (its neighbours and boltz_fill_boundary own them).
constexpr int kTrCells = 8;

template <int N>
__global__ void __launch_bounds__(256)
k_transport(const double* __restrict__ f, const double* __restrict__ base, double alpha, double* __restrict__ out,
            long long ncl, const double* __restrict__ x, const double* __restrict__ dx, double dt, int wl, int wr,
            double dv, int peer, double* __restrict__ left_dst, double* __restrict__ right_dst, long long cb,
            long long ce) {
    constexpr int N3 = N * N * N;
    constexpr int P3 = N3 / 2;  // node pairs: a thread owns nodes 2p, 2p+1 (same v1: N is even)
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    // the launch covers interior rows [cb, ce) (the whole interior [2, ncl + 2) unless a
    // halo-overlapped stage splits it, boltz_transport_step_range)
    const long long c0 = cb + (long long)blockIdx.y * kTrCells;
    const long long c1 = c0 + kTrCells < ce ? c0 + kTrCells : ce;  // [c0, c1) interior
    // per-cell geometry of cells c0-1 .. c1 (slopes) and c0 .. c1-1 (dt/dx)
    __shared__ double s_r1[kTrCells + 2], s_r2[kTrCells + 2], s_r3[kTrCells + 2], s_h[kTrCells + 2];
    __shared__ double s_lam[kTrCells];
    for (int t = threadIdx.x; t < (int)(c1 - c0) + 2; t += blockDim.x) {
        const long long c = c0 - 1 + t;
        s_r1[t] = 1.0 / (x[c + 1] - x[c]);
        s_r2[t] = 1.0 / (x[c] - x[c - 1]);
        s_r3[t] = 1.0 / (x[c + 1] - x[c - 1]);
        s_h[t] = 0.5 * dx[c];
        if (t < (int)(c1 - c0)) s_lam[t] = dt / dx[c0 + t];
    }
    __syncthreads();
    if (p >= P3) return;
    const double2* F = reinterpret_cast<const double2*>(f);
    const double2* Bs = reinterpret_cast<const double2*>(base);
    double2* O = reinterpret_cast<double2*>(out);
    if (!peer) {  // ghost rows copied through (by the launch that owns the adjacent interior rows)
        if (blockIdx.y == 0 && cb == 2) {
            O[p] = F[p];
            O[P3 + p] = F[P3 + p];
        }
        if (c1 == ncl + 2) {
            O[(ncl + 2) * P3 + p] = F[(ncl + 2) * P3 + p];
            O[(ncl + 3) * P3 + p] = F[(ncl + 3) * P3 + p];
        }
    }
    const double v1 = dv * ((2 * p) / (N * N) - N / 2);
    // slope of cell c (window index t = c - c0 + 1) from f[c-1], f[c], f[c+1]
    auto slope = [&](long long c, double fm, double f0, double fp) {
        const int t = (int)(c - c0 + 1);
        double sl = minmod3((fp - f0) * s_r1[t], (f0 - fm) * s_r2[t], (fp - fm) * s_r3[t]);
        if (wl && (c == 1 || c == 2)) sl = 0.0;
        if (wr && (c == ncl + 2 || c == ncl + 1)) sl = 0.0;
        return sl;
    };
    auto slope2 = [&](long long c, double2 fm, double2 f0, double2 fp) {
        return make_double2(slope(c, fm.x, f0.x, fp.x), slope(c, fm.y, f0.y, fp.y));
    };
    // upwind flux through the face between cells c and c+1
    auto face = [&](long long c, double fa, double sa, double fb, double sb) {
        return v1 >= 0.0 ? v1 * (fa + s_h[c - c0 + 1] * sa) : v1 * (fb - s_h[c - c0 + 2] * sb);
    };
    auto face2 = [&](long long c, double2 fa, double2 sa, double2 fb, double2 sb) {
        return make_double2(face(c, fa.x, sa.x, fb.x, sb.x), face(c, fa.y, sa.y, fb.y, sb.y));
    };
    double2 fm1 = F[(c0 - 1) * P3 + p], f0 = F[c0 * P3 + p], fp1 = F[(c0 + 1) * P3 + p];
    double2 sm1 = slope2(c0 - 1, F[(c0 - 2) * P3 + p], fm1, f0);
    double2 s0 = slope2(c0, fm1, f0, fp1);
    double2 Fl = face2(c0 - 1, fm1, sm1, f0, s0);
    for (long long ce = c0; ce < c1; ++ce) {
        const double2 fp2 = F[(ce + 2) * P3 + p];
        const double2 sp1 = slope2(ce + 1, f0, fp1, fp2);
        const double2 Fr = face2(ce, f0, s0, fp1, sp1);
        const double lam = s_lam[ce - c0];
        double2 v = make_double2(f0.x - lam * (Fr.x - Fl.x), f0.y - lam * (Fr.y - Fl.y));
        if (base) {
            const double2 b = Bs[ce * P3 + p];
            v = make_double2(alpha * b.x + (1.0 - alpha) * v.x, alpha * b.y + (1.0 - alpha) * v.y);
        }
        O[ce * P3 + p] = v;
        if (left_dst && ce < 4) reinterpret_cast<double2*>(left_dst)[(ce - 2) * P3 + p] = v;
        if (right_dst && ce >= ncl) reinterpret_cast<double2*>(right_dst)[(ce - ncl) * P3 + p] = v;
        f0 = fp1;
        fp1 = fp2;
        s0 = sp1;
        Fl = Fr;
    }
}

// the collision step's half of the fused exchange: cells 0,1 and n-2,n-1 of a
// rank's interior batch -> the neighbours' ghosts (same addressing as above)
template <int N>
__global__ void __launch_bounds__(256)
k_store_edges(const double* __restrict__ interior, long long n, double* __restrict__ left_dst,
              double* __restrict__ right_dst) {
    constexpr int N3 = N * N * N;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int e = blockIdx.y;  // 0,1: left edge cells; 2,3: right edge cells
    if (j >= N3) return;
    if (e < 2) {
        if (left_dst) left_dst[(size_t)e * N3 + j] = interior[(size_t)e * N3 + j];
    } else if (right_dst) {
        right_dst[(size_t)(e - 2) * N3 + j] = interior[(size_t)(n - 4 + e) * N3 + j];
    }
}

inline void launch_store_edges(int n, const double* interior, long long ncells, double* left_dst, double* right_dst,
                               cudaStream_t s) {
    switch (n) {
#define BOLTZ_SE(N)                                                                                  \
    case N: {                                                                                        \
        dim3 grid((N * N * N + 255) / 256, 4);                                                       \
        k_store_edges<N><<<grid, 256, 0, s>>>(interior, ncells, left_dst, right_dst);                \
    } break;
        BOLTZ_FOR_EACH_N(BOLTZ_SE)
#undef BOLTZ_SE
        default: break;
    }
}

// Boundary-flux ledger: acc[a] += coef * (F_a(right end face) - F_a(left end face))
// for the 5 collision invariants a (w, v1 w, v2 w, v3 w, |v|^2/2 w) -- the
// faces of the rank's first and last interior cells, the same values the FV
// step uses.  Summed over ranks, interior faces cancel exactly, so
//   ledger(t) - ledger(0) + acc == 0   up to round-off.
// One block of 256 threads, fixed-order tree reduction.
template <int N>
__global__ void __launch_bounds__(256)
k_end_flux(const double* __restrict__ f, long long ncl, const double* __restrict__ x, const double* __restrict__ dx,
           int wl, int wr, double dv, double coef, double* __restrict__ acc) {
    constexpr int N3 = N * N * N;
    const StencilCoef kl = stencil_coef(2, x, dx), kr = stencil_coef(ncl + 1, x, dx);
    double m[5] = {0, 0, 0, 0, 0};
    for (int j = threadIdx.x; j < N3; j += blockDim.x) {
        const int a1 = j / (N * N), a2 = (j / N) % N, a3 = j % N;
        const double v1 = dv * (a1 - N / 2), v2 = dv * (a2 - N / 2), v3 = dv * (a3 - N / 2);
        const double w = axis_coeff(N, a1) * axis_coeff(N, a2) * axis_coeff(N, a3) * dv * dv * dv;
        double fc, Fl, Fr, Gl, Gr;
        face_fluxes<N>(f, 2, j, ncl, kl, wl, wr, dv, fc, Fl, Gr);
        face_fluxes<N>(f, ncl + 1, j, ncl, kr, wl, wr, dv, fc, Gl, Fr);
        const double q = (Fr - Fl) * w;
        m[0] += q;
        m[1] += v1 * q;
        m[2] += v2 * q;
        m[3] += v3 * q;
        m[4] += 0.5 * (v1 * v1 + v2 * v2 + v3 * v3) * q;
    }
    __shared__ double red[5][256];
#pragma unroll
    for (int a = 0; a < 5; ++a) red[a][threadIdx.x] = m[a];
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s)
#pragma unroll
            for (int a = 0; a < 5; ++a) red[a][threadIdx.x] += red[a][threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x < 5) acc[threadIdx.x] += coef * red[threadIdx.x][0];
}

inline void launch_end_flux(int n, const double* f, long long ncl, const double* x, const double* dx, int wl, int wr,
                            double dv, double coef, double* acc, cudaStream_t s) {
    switch (n) {
#define BOLTZ_EF(N) \
    case N: k_end_flux<N><<<1, 256, 0, s>>>(f, ncl, x, dx, wl, wr, dv, coef, acc); break;
        BOLTZ_FOR_EACH_N(BOLTZ_EF)
#undef BOLTZ_EF
        default: break;
    }
}

// one block of kFillThreads threads; sigma_w written to sig[0]
constexpr int kFillThreads = 1024;  // one block: the wall's sigma_w is a whole-cell reduction

template <int N>
__global__ void __launch_bounds__(kFillThreads)
k_fill_boundary(double* __restrict__ f, long long ncl, const double* __restrict__ x, int side, int kind, double Tw,
                double vw0, double vw1, double vw2, double dv, double* __restrict__ sig) {
    constexpr int N3 = N * N * N;
    const long long g0 = side == 0 ? 1 : ncl + 2, g1 = side == 0 ? 0 : ncl + 3;
    const long long i0 = side == 0 ? 2 : ncl + 1, i1 = side == 0 ? 3 : ncl;
    double* G0 = f + g0 * N3;
    double* G1 = f + g1 * N3;
    const double* I0 = f + i0 * N3;
    const double* I1 = f + i1 * N3;
    if (kind == 0) {
        const double xa = x[i0], xb = x[i1];
        for (int j = threadIdx.x; j < N3; j += blockDim.x) {
            const double slope = (I0[j] - I1[j]) / (xa - xb);
            G0[j] = I0[j] + slope * (x[g0] - xa);
            G1[j] = I0[j] + slope * (x[g1] - xa);
        }
        if (threadIdx.x == 0) sig[0] = 0.0;
        return;
    }
    const double nrm = side == 0 ? 1.0 : -1.0;
    __shared__ double red[kFillThreads];
    double part = 0.0;
    for (int j = threadIdx.x; j < N3; j += blockDim.x) {
        const int a1 = j / (N * N), a2 = (j / N) % N, a3 = j % N;
        const double un = (dv * (a1 - N / 2) - vw0) * nrm;
        if (un <= 0.0) part += un * I0[j] * (axis_coeff(N, a1) * axis_coeff(N, a2) * axis_coeff(N, a3) * dv * dv * dv);
    }
    red[threadIdx.x] = part;
    __syncthreads();
    for (int w = kFillThreads / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    const double out = red[0];
    double sw = -sqrt(2.0 * kPi / Tw) * out;
    double norm = sw / pow(2.0 * kPi * Tw, 1.5);
    if (kind == 2) {
        // extension (not in the reference): discrete flux balance -- the wall
        // Maxwellian's lattice influx equals the lattice outflux (FV flux velocity v1)
        __syncthreads();
        double in = 0.0;
        for (int j = threadIdx.x; j < N3; j += blockDim.x) {
            const int a1 = j / (N * N), a2 = (j / N) % N, a3 = j % N;
            const double c1 = dv * (a1 - N / 2) - vw0, c2 = dv * (a2 - N / 2) - vw1, c3 = dv * (a3 - N / 2) - vw2;
            if (c1 * nrm > 0.0)
                in += dv * (a1 - N / 2) * nrm * exp(-(c1 * c1 + c2 * c2 + c3 * c3) / (2.0 * Tw)) *
                      (axis_coeff(N, a1) * axis_coeff(N, a2) * axis_coeff(N, a3) * dv * dv * dv);
        }
        red[threadIdx.x] = in;
        __syncthreads();
        for (int w = kFillThreads / 2; w > 0; w >>= 1) {
            if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
            __syncthreads();
        }
        norm = red[0] > 0.0 ? -out / red[0] : 0.0;
        sw = norm * pow(2.0 * kPi * Tw, 1.5);
    }
    for (int j = threadIdx.x; j < N3; j += blockDim.x) {
        const int a1 = j / (N * N), a2 = (j / N) % N, a3 = j % N;
        const double c1 = dv * (a1 - N / 2) - vw0, c2 = dv * (a2 - N / 2) - vw1, c3 = dv * (a3 - N / 2) - vw2;
        const double val = (c1 * nrm > 0.0) ? norm * exp(-(c1 * c1 + c2 * c2 + c3 * c3) / (2.0 * Tw)) : 0.0;
        G0[j] = val;
        G1[j] = val;
    }
    if (threadIdx.x == 0) sig[0] = sw;
}

inline void launch_transport(int n, const double* f, const double* base, double alpha, double* out, long long ncl,
                             const double* x, const double* dx, double dt, int wl, int wr, double dv,
                             cudaStream_t s, int peer = 0, double* left_dst = nullptr,
                             double* right_dst = nullptr, long long cb = 2, long long ce = -1) {
    if (ce < 0) ce = ncl + 2;
    if (ce <= cb) return;
    switch (n) {
#define BOLTZ_TR(N)                                                                                        \
    case N: {                                                                                              \
        dim3 grid((N * N * N / 2 + 255) / 256, (unsigned)((ce - cb + kTrCells - 1) / kTrCells));          \
        k_transport<N><<<grid, 256, 0, s>>>(f, base, alpha, out, ncl, x, dx, dt, wl, wr, dv, peer, left_dst, \
                                            right_dst, cb, ce);                                            \
    } break;
        BOLTZ_FOR_EACH_N(BOLTZ_TR)
#undef BOLTZ_TR
        default: break;
    }
}

inline void launch_fill_boundary(int n, double* f, long long ncl, const double* x, int side, int kind, double Tw,
                                 double vw0, double vw1, double vw2, double dv, double* sig, cudaStream_t s) {
    switch (n) {
#define BOLTZ_FB(N) \
    case N: k_fill_boundary<N><<<1, kFillThreads, 0, s>>>(f, ncl, x, side, kind, Tw, vw0, vw1, vw2, dv, sig); break;
        BOLTZ_FOR_EACH_N(BOLTZ_FB)
#undef BOLTZ_FB
        default: break;
    }
}

}  // namespace boltz_gpu

namespace boltz_gpu {

// compute_moments for a batch of cells in the user layout:
// out[c] = {rho, rho V1, rho V2, rho V3, rho e, T, H} with rho e = 1/2 sum |v|^2 f w,
// T = (2 rho e / rho - |V|^2) / 3, H = sum_{f>0} f log f w.  One block per
// cell, fixed-order tree reduction (deterministic).
template <int N>
__global__ void __launch_bounds__(256) k_moments(const double* __restrict__ f, double* __restrict__ out, double dv) {
    constexpr int N3 = N * N * N;
    const long long cell = blockIdx.x;
    const double* fc = f + (size_t)cell * N3;
    double m[6] = {0, 0, 0, 0, 0, 0};
    const double dv3 = dv * dv * dv;
    for (int j = threadIdx.x; j < N3; j += blockDim.x) {
        const int a1 = j / (N * N), a2 = (j / N) % N, a3 = j % N;
        const double v1 = dv * (a1 - N / 2), v2 = dv * (a2 - N / 2), v3 = dv * (a3 - N / 2);
        const double w = axis_coeff(N, a1) * axis_coeff(N, a2) * axis_coeff(N, a3) * dv3;
        const double x = fc[j], q = x * w;
        m[0] += q;
        m[1] += v1 * q;
        m[2] += v2 * q;
        m[3] += v3 * q;
        m[4] += (v1 * v1 + v2 * v2 + v3 * v3) * q;
        if (x > 0) m[5] += x * log(x) * w;
    }
    __shared__ double red[6][256];
#pragma unroll
    for (int a = 0; a < 6; ++a) red[a][threadIdx.x] = m[a];
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s)
#pragma unroll
            for (int a = 0; a < 6; ++a) red[a][threadIdx.x] += red[a][threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double rho = red[0][0];
        double* o = out + cell * 7;
        o[0] = rho;
        o[1] = red[1][0];
        o[2] = red[2][0];
        o[3] = red[3][0];
        o[4] = 0.5 * red[4][0];
        double T = 0.0;
        if (rho > 0) {
            const double V2 = (o[1] * o[1] + o[2] * o[2] + o[3] * o[3]) / (rho * rho);
            T = (2.0 * o[4] / rho - V2) / 3.0;
        }
        o[5] = T;
        o[6] = red[5][0];
    }
}

// marginal_distribution (SPEC.md cli_io/scenario module): g(v1_i) =
// sum_{i2,i3} f c(i2) c(i3) dv^2, N values per cell.  One block per cell, one
// warp per v1 plane; fixed lane-stride + xor-tree order (deterministic).
template <int N>
__global__ void __launch_bounds__(256) k_marginal(const double* __restrict__ f, double* __restrict__ g, double dv) {
    constexpr int N2 = N * N;
    const long long cell = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i1 = w; i1 < N; i1 += 8) {
        const double* p = f + ((size_t)cell * N + i1) * N2;
        double s = 0.0;
        for (int j = lane; j < N2; j += 32) s += p[j] * axis_coeff(N, j / N) * axis_coeff(N, j % N);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) g[(size_t)cell * N + i1] = s * dv * dv;
    }
}

inline void launch_marginal(int n, const double* f, double* g, long long ncells, double dv, cudaStream_t s) {
    switch (n) {
#define BOLTZ_MA(N) \
    case N: k_marginal<N><<<(unsigned)ncells, 256, 0, s>>>(f, g, dv); break;
        BOLTZ_FOR_EACH_N(BOLTZ_MA)
#undef BOLTZ_MA
        default: break;
    }
}

inline void launch_moments(int n, const double* f, double* out, long long ncells, double dv, cudaStream_t s) {
    switch (n) {
#define BOLTZ_MO(N) \
    case N: k_moments<N><<<(unsigned)ncells, 256, 0, s>>>(f, out, dv); break;
        BOLTZ_FOR_EACH_N(BOLTZ_MO)
#undef BOLTZ_MO
        default: break;
    }
}

}  // namespace boltz_gpu
