/*
 * boltz_oracle.c -- CPU ORACLE (TEST INFRASTRUCTURE ONLY).
 *
 * A plain-C restatement of the reference's conservative spectral Boltzmann
 * collision path (arXiv 1301.4195; reference tree: PAPER.md + SPEC.md + the
 * three headers and one .cpp under proj/).  It exists to CHECK the CUDA path
 * in paper_1301_4195_b200/csrc; nothing in the product may link or call it.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg load it.
 *
 * Parity status:
 *   - velocity grid: PINNED against the reference's own velocity_grid.cpp,
 *     compiled from /root/reference by oracle/Makefile into oracle/_ref and
 *     frozen as tests/golden/grid_ref.json.
 *   - transforms / weights / collision / projection / transport: the
 *     reference ships no implementation (collision.cpp, fourier.cpp, ... are
 *     absent, CMakeLists.txt:22-33) and no golden vectors; FFTW (unpinned
 *     version) is absent.  These are pinned only to SPEC.md's known-answer
 *     tests (direct-sum DFT, naive-loop qhat, quadrature-vs-closed-form
 *     weights, conservation/idempotence) -- "parity partially unpinned".
 *
 * Everything is naive, deterministic and in lexicographic order
 * (SPEC.md:233).  The only parallel code is bo_evaluate_qhat_omp, the
 * reference's own OpenMP map over zeta_k,
 * kept solely to time the CPU baseline.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define BO_PI 3.14159265358979323846264338327950288

/* ------------------------------------------------------------------ */
/* velocity grid  (velocity_grid.hpp:17-47, velocity_grid.cpp:11-32)   */
/* ------------------------------------------------------------------ */

/* returns 0, or 2 (ConfigError, errors.hpp:8-13) for odd N, N<4, L<=0 */
int bo_grid(int n, double L, double *dv, double *dzeta, double *v_nodes,
            double *zeta_nodes, double *axis_coeff) {
    if (n < 4 || n % 2 != 0) return 2;
    if (!(L > 0.0)) return 2;
    double h = 2.0 * L / n, dz = BO_PI / L;
    if (dv) *dv = h;
    if (dzeta) *dzeta = dz;
    for (int k = 0; k < n; ++k) {
        if (v_nodes) v_nodes[k] = h * (k - n / 2);
        if (zeta_nodes) zeta_nodes[k] = dz * (k - n / 2);
        if (axis_coeff) axis_coeff[k] = (k == 0 || k == n - 1) ? 0.5 : 1.0;
    }
    return 0;
}

static double axc(int n, int k) { return (k == 0 || k == n - 1) ? 0.5 : 1.0; }

/* ------------------------------------------------------------------ */
/* weights                         */
/* ------------------------------------------------------------------ */

/* h(x) = (x sin x + cos x - 1)/x^2 = int_0^1 t cos(xt) dt */
static double bo_h(double x) {
    double ax = fabs(x);
    if (ax < 1.0) {
        double x2 = x * x, term = 1.0, s = 0.0; /* term = (-1)^n x^2n/(2n)! */
        for (int n = 0; n < 24; ++n) {
            s += term / (2.0 * n + 2.0);
            term *= -x2 / ((2.0 * n + 1.0) * (2.0 * n + 2.0));
        }
        return s;
    }
    return (x * sin(x) + cos(x) - 1.0) / (x * x);
}

/* j1(x) = int_0^1 t^3 sinc(xt) dt = ((2-x^2)cos x + 2x sin x - 2)/x^4 */
static double bo_j1(double x) {
    double ax = fabs(x);
    if (ax < 1.5) {
        double x2 = x * x, term = 1.0, s = 0.0; /* (-1)^n x^2n/(2n+1)! */
        for (int n = 0; n < 28; ++n) {
            s += term / (2.0 * n + 4.0);
            term *= -x2 / ((2.0 * n + 2.0) * (2.0 * n + 3.0));
        }
        return s;
    }
    double x2 = x * x;
    return ((2.0 - x2) * cos(x) + 2.0 * x * sin(x) - 2.0) / (x2 * x2);
}

/* j0(x) = int_0^1 t^2 sinc(xt) dt = (sin x - x cos x)/x^3 */
static double bo_j0(double x) {
    double ax = fabs(x);
    if (ax < 1.0) {
        double x2 = x * x, term = 1.0, s = 0.0;
        for (int n = 0; n < 24; ++n) {
            s += term / (2.0 * n + 3.0);
            term *= -x2 / ((2.0 * n + 2.0) * (2.0 * n + 3.0));
        }
        return s;
    }
    return (sin(x) - x * cos(x)) / (x * x * x);
}

static double bo_sinc(double x) {
    double ax = fabs(x);
    if (ax < 1e-3) {
        double x2 = x * x;
        return 1.0 - x2 / 6.0 * (1.0 - x2 / 20.0 * (1.0 - x2 / 42.0));
    }
    return sin(x) / x;
}

/*
 * Closed form of PAPER.md:181-185 for lambda in {0,1}, with p=a-b, q=a+b
 * and every removable singularity
 * replaced by its limit.  a = beta|zeta|/2, b = |xi - beta zeta/2|, c=|xi|.
 * p is formed as (a^2-b^2)/(a+b) with a^2-b^2 = beta xi.zeta - |xi|^2, so an
 * exact a=b gives p=0 instead of a rounding residue.
 * Returns NAN for lambda not in {0,1} ("reject").
 */
double bo_weight_closed_form(double lambda, double beta, double r0,
                             const double xi[3], const double zeta[3]) {
    double zz = 0, xx = 0, xz = 0, bb = 0;
    for (int i = 0; i < 3; ++i) {
        double w = xi[i] - 0.5 * beta * zeta[i];
        zz += zeta[i] * zeta[i];
        xx += xi[i] * xi[i];
        xz += xi[i] * zeta[i];
        bb += w * w;
    }
    double a = 0.5 * beta * sqrt(zz), b = sqrt(bb), c = sqrt(xx);
    const double C0 = 4.0 * BO_PI / pow(2.0 * BO_PI, 1.5);
    double T1, T2;
    if (lambda == 1.0) {
        double r2 = r0 * r0, r4 = r2 * r2;
        if (a == 0.0 && b == 0.0) T1 = 0.25 * r4;
        else if (a == 0.0) T1 = r4 * bo_j1(b * r0);
        else if (b == 0.0) T1 = r4 * bo_j1(a * r0);
        else {
            double p = (beta * xz - xx) / (a + b), q = a + b;
            T1 = r2 * (bo_h(p * r0) - bo_h(q * r0)) / (2.0 * a * b);
        }
        T2 = r4 * bo_j1(c * r0);
    } else if (lambda == 0.0) {
        double r3 = r0 * r0 * r0;
        if (a == 0.0 && b == 0.0) T1 = r3 / 3.0;
        else if (a == 0.0) T1 = r3 * bo_j0(b * r0);
        else if (b == 0.0) T1 = r3 * bo_j0(a * r0);
        else {
            double p = (beta * xz - xx) / (a + b), q = a + b;
            T1 = r0 * (bo_sinc(p * r0) - bo_sinc(q * r0)) / (2.0 * a * b);
        }
        T2 = r3 * bo_j0(c * r0);
    } else {
        return NAN;
    }
    return C0 * (T1 - T2);
}

/* Gauss-Legendre nodes/weights on [-1,1] (Newton on P_n) */
static void bo_gauss_legendre(int n, double *x, double *w) {
    for (int i = 0; i < (n + 1) / 2; ++i) {
        double z = cos(BO_PI * (i + 0.75) / (n + 0.5)), pp = 0;
        for (int it = 0; it < 100; ++it) {
            double p1 = 1.0, p2 = 0.0;
            for (int j = 1; j <= n; ++j) {
                double p3 = p2;
                p2 = p1;
                p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
            }
            pp = n * (z * p1 - p2) / (z * z - 1.0);
            double z1 = z;
            z = z1 - p1 / pp;
            if (fabs(z - z1) < 1e-16) break;
        }
        x[i] = -z;
        x[n - 1 - i] = z;
        w[i] = w[n - 1 - i] = 2.0 / ((1.0 - z * z) * pp * pp);
    }
}

/*
 * weight_quadrature: composite Gauss-Legendre, `panels`
 * panels of 16 nodes on [0, r0], of r^{lambda+2}[sinc(a r)sinc(b r)-sinc(c r)].
 */
double bo_weight_quadrature(double lambda, double beta, double r0,
                            const double xi[3], const double zeta[3], int panels) {
    double zz = 0, xx = 0, bb = 0;
    for (int i = 0; i < 3; ++i) {
        double w = xi[i] - 0.5 * beta * zeta[i];
        zz += zeta[i] * zeta[i];
        xx += xi[i] * xi[i];
        bb += w * w;
    }
    double a = 0.5 * beta * sqrt(zz), b = sqrt(bb), c = sqrt(xx);
    double gx[16], gw[16];
    bo_gauss_legendre(16, gx, gw);
    double h = r0 / panels, s = 0.0;
    for (int p = 0; p < panels; ++p) {
        double lo = p * h;
        for (int i = 0; i < 16; ++i) {
            double r = lo + 0.5 * h * (gx[i] + 1.0);
            double f = pow(r, lambda + 2.0) *
                       (bo_sinc(a * r) * bo_sinc(b * r) - bo_sinc(c * r));
            s += 0.5 * h * gw[i] * f;
        }
    }
    return 4.0 * BO_PI / pow(2.0 * BO_PI, 1.5) * s;
}

/*
 * generate_table: zeta-major G[k][m], k the
 * flat zeta index, m the flat xi index, N^6 doubles.  Closed form for
 * lambda in {0,1}, quadrature (`panels`) otherwise.  A pure parallel map,
 * bit-identical for any thread count.
 */
void bo_generate_table(int n, double L, double lambda, double beta, double r0,
                       int panels, double *G, int nthreads) {
    const int64_t M = (int64_t)n * n * n;
    const double dz = BO_PI / L;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t k = 0; k < M; ++k) {
        double zeta[3] = {dz * ((int)(k / (n * n)) - n / 2),
                          dz * ((int)((k / n) % n) - n / 2),
                          dz * ((int)(k % n) - n / 2)};
        for (int64_t m = 0; m < M; ++m) {
            double xi[3] = {dz * ((int)(m / (n * n)) - n / 2),
                            dz * ((int)((m / n) % n) - n / 2),
                            dz * ((int)(m % n) - n / 2)};
            G[k * M + m] = (lambda == 0.0 || lambda == 1.0)
                               ? bo_weight_closed_form(lambda, beta, r0, xi, zeta)
                               : bo_weight_quadrature(lambda, beta, r0, xi, zeta, panels);
        }
    }
}

/* ------------------------------------------------------------------ */
/* transforms  (fourier.hpp:11-22,36-41)                */
/* complex arrays are interleaved (re, im) doubles                     */
/* ------------------------------------------------------------------ */

/* apply a 1D N-point matrix E (complex, [k][m]) along one axis, in place */
static void bo_axis_apply(int n, double *z, const double *E, int axis) {
    int64_t stride = axis == 0 ? (int64_t)n * n : (axis == 1 ? n : 1);
    double *tr = malloc(sizeof(double) * 2 * n);
    for (int64_t base = 0; base < (int64_t)n * n * n; ++base) {
        int ia = (int)((base / stride) % n);
        if (ia != 0) continue; /* visit each line once, at its index-0 element */
        for (int k = 0; k < n; ++k) {
            double sr = 0, si = 0;
            for (int m = 0; m < n; ++m) {
                const double *x = z + 2 * (base + m * stride);
                double er = E[2 * (k * n + m)], ei = E[2 * (k * n + m) + 1];
                sr += er * x[0] - ei * x[1];
                si += er * x[1] + ei * x[0];
            }
            tr[2 * k] = sr;
            tr[2 * k + 1] = si;
        }
        for (int k = 0; k < n; ++k) {
            z[2 * (base + k * stride)] = tr[2 * k];
            z[2 * (base + k * stride) + 1] = tr[2 * k + 1];
        }
    }
    free(tr);
}

/*
 * forward (fourier.hpp:11-12): fhat(zeta_k) = (dv/sqrt(2pi))^3 sum_m c_m f(v_m)
 * e^{-i zeta_k . v_m}.  Evaluated as the literal separable direct sum (one
 * 1D DFT matrix per axis built from cos/sin of zeta_k v_m), i.e. WITHOUT the
 * index-space phase trick, so it independently checks the GPU's
 * phase-wrapped FFT (fourier.hpp:19-22).
 */
void bo_forward(int n, double L, const double *f, double *fhat) {
    const int64_t M = (int64_t)n * n * n;
    double dv = 2.0 * L / n, dz = BO_PI / L;
    double *E = malloc(sizeof(double) * 2 * n * n);
    for (int k = 0; k < n; ++k)
        for (int m = 0; m < n; ++m) {
            double ph = (dz * (k - n / 2)) * (dv * (m - n / 2));
            E[2 * (k * n + m)] = cos(ph);
            E[2 * (k * n + m) + 1] = -sin(ph);
        }
    double s = dv / sqrt(2.0 * BO_PI);
    double scale = s * s * s;
    for (int64_t i = 0; i < M; ++i) {
        int i1 = (int)(i / (n * n)), i2 = (int)((i / n) % n), i3 = (int)(i % n);
        fhat[2 * i] = f[i] * axc(n, i1) * axc(n, i2) * axc(n, i3);
        fhat[2 * i + 1] = 0.0;
    }
    for (int ax = 2; ax >= 0; --ax) bo_axis_apply(n, fhat, E, ax);
    for (int64_t i = 0; i < 2 * M; ++i) fhat[i] *= scale;
    free(E);
}

/*
 * inverse (fourier.hpp:15-17,38-41): f(v_k) = Re (dzeta/sqrt(2pi))^3 sum_m
 * g(zeta_m) e^{+i v_k . zeta_m}, a plain lattice sum (no trapezoid weights;
 * header convention).  *max_imag = max |Im|.
 */
void bo_inverse(int n, double L, const double *g, double *f, double *max_imag) {
    const int64_t M = (int64_t)n * n * n;
    double dv = 2.0 * L / n, dz = BO_PI / L;
    double *E = malloc(sizeof(double) * 2 * n * n);
    for (int k = 0; k < n; ++k)
        for (int m = 0; m < n; ++m) {
            double ph = (dv * (k - n / 2)) * (dz * (m - n / 2));
            E[2 * (k * n + m)] = cos(ph);
            E[2 * (k * n + m) + 1] = sin(ph);
        }
    double *z = malloc(sizeof(double) * 2 * M);
    memcpy(z, g, sizeof(double) * 2 * M);
    for (int ax = 2; ax >= 0; --ax) bo_axis_apply(n, z, E, ax);
    double s = dz / sqrt(2.0 * BO_PI);
    double scale = s * s * s, mi = 0.0;
    for (int64_t i = 0; i < M; ++i) {
        f[i] = scale * z[2 * i];
        double im = fabs(scale * z[2 * i + 1]);
        if (im > mi) mi = im;
    }
    if (max_imag) *max_imag = mi;
    free(z);
    free(E);
}

/* ------------------------------------------------------------------ */
/* collision                      */
/* ------------------------------------------------------------------ */

/* one output zeta_k of evaluate_qhat, naive lexicographic order */
static void bo_qhat_one(int n, double L, const double *G, const double *fhat,
                        int64_t k, double *out) {
    const int64_t M = (int64_t)n * n * n;
    double dz = BO_PI / L, w3 = dz * dz * dz;
    int k1 = (int)(k / (n * n)), k2 = (int)((k / n) % n), k3 = (int)(k % n);
    const double *Gk = G + k * M;
    double sr = 0.0, si = 0.0;
    for (int m1 = 0; m1 < n; ++m1) {
        int s1 = k1 - m1 + n / 2;
        if (s1 < 0 || s1 >= n) continue;
        for (int m2 = 0; m2 < n; ++m2) {
            int s2 = k2 - m2 + n / 2;
            if (s2 < 0 || s2 >= n) continue;
            for (int m3 = 0; m3 < n; ++m3) {
                int s3 = k3 - m3 + n / 2;
                if (s3 < 0 || s3 >= n) continue; /* off-lattice: fhat = 0 */
                int64_t m = ((int64_t)m1 * n + m2) * n + m3;
                int64_t s = ((int64_t)s1 * n + s2) * n + s3;
                double om = axc(n, m1) * axc(n, m2) * axc(n, m3) * w3;
                double gw = Gk[m] * om;
                double ar = fhat[2 * m], ai = fhat[2 * m + 1];
                double br = fhat[2 * s], bi = fhat[2 * s + 1];
                sr += gw * (ar * br - ai * bi);
                si += gw * (ar * bi + ai * br);
            }
        }
    }
    out[0] = sr;
    out[1] = si;
}

/*
 * evaluate_qhat: Qhat(zeta_k) = sum_m G(xi_m,zeta_k)
 * fhat(xi_m) fhat(zeta_k - xi_m) omega_m, shifted index k-m+N/2 per axis,
 * kept only in [0,N-1].
 */
void bo_evaluate_qhat(int n, double L, const double *G, const double *fhat,
                      double *qhat) {
    const int64_t M = (int64_t)n * n * n;
    for (int64_t k = 0; k < M; ++k) bo_qhat_one(n, L, G, fhat, k, qhat + 2 * k);
}

/* the reference's parallelisation: OpenMP map over zeta_k */
void bo_evaluate_qhat_omp(int n, double L, const double *G, const double *fhat,
                          double *qhat, int nthreads) {
    const int64_t M = (int64_t)n * n * n;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t k = 0; k < M; ++k) bo_qhat_one(n, L, G, fhat, k, qhat + 2 * k);
}

/* 5x5 Gram matrix C C^T of ConservationOperator */
static void bo_constraint_row(int n, double L, int64_t j, double row[5]) {
    double dv = 2.0 * L / n;
    int i1 = (int)(j / (n * n)), i2 = (int)((j / n) % n), i3 = (int)(j % n);
    double w = axc(n, i1) * axc(n, i2) * axc(n, i3) * dv * dv * dv;
    double v1 = dv * (i1 - n / 2), v2 = dv * (i2 - n / 2), v3 = dv * (i3 - n / 2);
    row[0] = w;
    row[1] = v1 * w;
    row[2] = v2 * w;
    row[3] = v3 * w;
    row[4] = (v1 * v1 + v2 * v2 + v3 * v3) * w;
}

/*
 * conserve: Q = Qt - C^T (C C^T)^{-1} C Qt, the Lagrange
 * solution (the paper's printed Qt + C(CC^T)^{-1}CQt, is
 * dimensionally inconsistent).  Cholesky solve.
 */
void bo_conserve(int n, double L, const double *qt, double *q) {
    const int64_t M = (int64_t)n * n * n;
    double A[5][5] = {{0}}, r[5] = {0}, row[5];
    for (int64_t j = 0; j < M; ++j) {
        bo_constraint_row(n, L, j, row);
        for (int a = 0; a < 5; ++a) {
            r[a] += row[a] * qt[j];
            for (int b = 0; b < 5; ++b) A[a][b] += row[a] * row[b];
        }
    }
    /* Cholesky A = R R^T */
    double R[5][5] = {{0}};
    for (int i = 0; i < 5; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = A[i][j];
            for (int k = 0; k < j; ++k) s -= R[i][k] * R[j][k];
            R[i][j] = (i == j) ? sqrt(s) : s / R[j][j];
        }
    double y[5], lam[5];
    for (int i = 0; i < 5; ++i) {
        double s = r[i];
        for (int k = 0; k < i; ++k) s -= R[i][k] * y[k];
        y[i] = s / R[i][i];
    }
    for (int i = 4; i >= 0; --i) {
        double s = y[i];
        for (int k = i + 1; k < 5; ++k) s -= R[k][i] * lam[k];
        lam[i] = s / R[i][i];
    }
    for (int64_t j = 0; j < M; ++j) {
        bo_constraint_row(n, L, j, row);
        double c = 0;
        for (int a = 0; a < 5; ++a) c += row[a] * lam[a];
        q[j] = qt[j] - c;
    }
}

/*
 * collide: (1/eps) P_N(inverse(evaluate_qhat(forward(f)))).
 * Returns 0, or 4 (NumericError, errors.hpp:33-35) on non-finite input.
 * `nthreads` > 0 selects the OpenMP qhat (baseline timing); 0 = serial.
 */
int bo_collide(int n, double L, const double *G, const double *f, double eps,
               double *q, double *max_imag, int nthreads) {
    const int64_t M = (int64_t)n * n * n;
    for (int64_t i = 0; i < M; ++i)
        if (!isfinite(f[i])) return 4;
    double *fh = malloc(sizeof(double) * 2 * M), *qh = malloc(sizeof(double) * 2 * M);
    double *qt = malloc(sizeof(double) * M);
    bo_forward(n, L, f, fh);
    if (nthreads > 0) bo_evaluate_qhat_omp(n, L, G, fh, qh, nthreads);
    else bo_evaluate_qhat(n, L, G, fh, qh);
    bo_inverse(n, L, qh, qt, max_imag);
    bo_conserve(n, L, qt, q);
    for (int64_t i = 0; i < M; ++i) q[i] /= eps;
    free(fh);
    free(qh);
    free(qt);
    return 0;
}

/*
 * collision_rk2: midpoint RK2 per cell,
 * f* = f + (dt/2) collide(f); f <- f + dt collide(f*).  In place over
 * `ncells` consecutive N^3 blocks.  Returns 0 or 4.
 */
int bo_collision_rk2(int n, double L, const double *G, double *f, int64_t ncells,
                     double dt, double eps, int nthreads) {
    const int64_t M = (int64_t)n * n * n;
    double *fs = malloc(sizeof(double) * M), *q = malloc(sizeof(double) * M);
    int rc = 0;
    for (int64_t c = 0; c < ncells && rc == 0; ++c) {
        double *fc = f + c * M;
        rc = bo_collide(n, L, G, fc, eps, q, NULL, nthreads);
        if (rc) break;
        for (int64_t i = 0; i < M; ++i) fs[i] = fc[i] + 0.5 * dt * q[i];
        rc = bo_collide(n, L, G, fs, eps, q, NULL, nthreads);
        if (rc) break;
        for (int64_t i = 0; i < M; ++i) fc[i] += dt * q[i];
        for (int64_t i = 0; i < M; ++i)
            if (!isfinite(fc[i])) rc = 4;
    }
    free(fs);
    free(q);
    return rc;
}

/* ------------------------------------------------------------------ */
/* moments & scenarios                     */
/* out = {rho, rhoV1, rhoV2, rhoV3, rho e, T, H}                       */
/* ------------------------------------------------------------------ */
void bo_moments(int n, double L, const double *f, double out[7]) {
    const int64_t M = (int64_t)n * n * n;
    double dv = 2.0 * L / n, m[5] = {0}, H = 0, row[5];
    for (int64_t j = 0; j < M; ++j) {
        bo_constraint_row(n, L, j, row);
        for (int a = 0; a < 5; ++a) m[a] += row[a] * f[j];
        if (f[j] > 0) H += f[j] * log(f[j]) * row[0];
    }
    (void)dv;
    double rho = m[0];
    out[0] = rho;
    out[1] = m[1];
    out[2] = m[2];
    out[3] = m[3];
    out[4] = 0.5 * m[4];
    if (rho > 0) {
        double V2 = (m[1] * m[1] + m[2] * m[2] + m[3] * m[3]) / (rho * rho);
        out[5] = (2.0 * out[4] / rho - V2) / 3.0;
    } else {
        out[5] = 0.0;
    }
    out[6] = H;
}

/* marginal_distribution (SPEC.md "[OP] marginal_distribution", cli/scenario
 * module): g(v1_i) = sum_{i2,i3} f(i,i2,i3) c(i2) c(i3) dv^2. */
void bo_marginal(int n, double L, const double *f, double *g) {
    const double dv = 2.0 * L / n;
    for (int i1 = 0; i1 < n; ++i1) {
        double s = 0.0;
        for (int i2 = 0; i2 < n; ++i2)
            for (int i3 = 0; i3 < n; ++i3) s += f[((int64_t)i1 * n + i2) * n + i3] * axc(n, i2) * axc(n, i3);
        g[i1] = s * dv * dv;
    }
}

void bo_maxwellian(int n, double L, double rho, const double V[3], double T,
                   double *f) {
    double dv = 2.0 * L / n;
    double norm = rho / pow(2.0 * BO_PI * T, 1.5);
    for (int i1 = 0; i1 < n; ++i1)
        for (int i2 = 0; i2 < n; ++i2)
            for (int i3 = 0; i3 < n; ++i3) {
                double a = dv * (i1 - n / 2) - V[0], b = dv * (i2 - n / 2) - V[1],
                       c = dv * (i3 - n / 2) - V[2];
                f[((int64_t)i1 * n + i2) * n + i3] =
                    norm * exp(-(a * a + b * b + c * c) / (2.0 * T));
            }
}

/* ------------------------------------------------------------------ */
/* transport                      */
/* ------------------------------------------------------------------ */

double bo_minmod3(double a, double b, double c) {
    if (a > 0 && b > 0 && c > 0) return fmin(a, fmin(b, c));
    if (a < 0 && b < 0 && c < 0) return fmax(a, fmax(b, c));
    return 0.0;
}

/*
 * Fill the two ghost cells at one physical end.
 * field: (ncl+4) x M, interior at 2..ncl+1.  side 0 = left, 1 = right.
 * kind 0 = linear extrapolation from the two nearest interior cells
 *           using ghost centres xg[2] and interior centres;
 * kind 1 = diffuse wall with T_w, V_w(3);
 *          returns sigma_w through *sigma.
 * x_ext: centres of all ncl+4 (ghost+interior) cells of this field.
 */
void bo_fill_boundary(int n, double L, double *field, int64_t ncl,
                      const double *x_ext, int side, int kind, double Tw,
                      const double Vw[3], double *sigma) {
    const int64_t M = (int64_t)n * n * n;
    int64_t g0, g1, i0, i1; /* g0 adjacent ghost, g1 outer ghost; i0 adjacent interior */
    if (side == 0) { g0 = 1; g1 = 0; i0 = 2; i1 = 3; }
    else { g0 = ncl + 2; g1 = ncl + 3; i0 = ncl + 1; i1 = ncl; }
    double *G0 = field + g0 * M, *G1 = field + g1 * M;
    const double *I0 = field + i0 * M, *I1 = field + i1 * M;
    if (kind == 0) {
        double xa = x_ext[i0], xb = x_ext[i1];
        for (int64_t j = 0; j < M; ++j) {
            double slope = (I0[j] - I1[j]) / (xa - xb);
            G0[j] = I0[j] + slope * (x_ext[g0] - xa);
            G1[j] = I0[j] + slope * (x_ext[g1] - xa);
        }
        if (sigma) *sigma = 0.0;
        return;
    }
    /* wall: inward normal +e1 at the left end, -e1 at the right end */
    double nrm = side == 0 ? 1.0 : -1.0, dv = 2.0 * L / n, sw = 0.0;
    for (int64_t j = 0; j < M; ++j) {
        int a1 = (int)(j / (n * n)), a2 = (int)((j / n) % n), a3 = (int)(j % n);
        double un = (dv * (a1 - n / 2) - Vw[0]) * nrm;
        if (un <= 0.0) { /* outgoing (towards the wall) incl. grazing */
            double w = axc(n, a1) * axc(n, a2) * axc(n, a3) * dv * dv * dv;
            sw += un * I0[j] * w;
        }
    }
    double norm;
    if (kind == 2) {
        /* extension (not in the reference): discrete flux balance -- scale the
         * wall Maxwellian so that its lattice influx equals the lattice outflux
         * (v1 here is the FV flux velocity; zero net mass flux up to round-off) */
        double in = 0.0;
        for (int64_t j = 0; j < M; ++j) {
            int a1 = (int)(j / (n * n)), a2 = (int)((j / n) % n), a3 = (int)(j % n);
            double c1 = dv * (a1 - n / 2) - Vw[0], c2 = dv * (a2 - n / 2) - Vw[1], c3 = dv * (a3 - n / 2) - Vw[2];
            if (c1 * nrm > 0.0)
                in += dv * (a1 - n / 2) * nrm * exp(-(c1 * c1 + c2 * c2 + c3 * c3) / (2.0 * Tw)) *
                      (axc(n, a1) * axc(n, a2) * axc(n, a3) * dv * dv * dv);
        }
        norm = in > 0.0 ? -sw / in : 0.0;
        sw = norm * pow(2.0 * BO_PI * Tw, 1.5);
    } else {
        sw = -sqrt(2.0 * BO_PI / Tw) * sw;
        norm = sw / pow(2.0 * BO_PI * Tw, 1.5);
    }
    for (int64_t j = 0; j < M; ++j) {
        int a1 = (int)(j / (n * n)), a2 = (int)((j / n) % n), a3 = (int)(j % n);
        double c1 = dv * (a1 - n / 2) - Vw[0], c2 = dv * (a2 - n / 2) - Vw[1],
               c3 = dv * (a3 - n / 2) - Vw[2];
        double val = (c1 * nrm > 0.0) ? norm * exp(-(c1 * c1 + c2 * c2 + c3 * c3) / (2.0 * Tw)) : 0.0;
        G0[j] = val;
        G1[j] = val;
    }
    if (sigma) *sigma = sw;
}

/*
 * transport_step: one explicit FV step of
 * f_t + v1 f_x = 0 on the (ncl+4)-cell field with ghosts already filled.
 * x_ext/dx_ext: centres/widths of all ncl+4 cells.  wall_left/wall_right:
 * 1 if that end is a wall (zero slope in the ghost and the wall-adjacent
 * interior cell).  Writes the updated interior into out
 * (same layout; ghosts copied through).  Per-node flux F_{j+1/2} per
 * PAPER.md:288-291 with each cell's own half width.
 */
void bo_transport_step(int n, double L, const double *field, double *out,
                       int64_t ncl, const double *x_ext, const double *dx_ext,
                       double dt, int wall_left, int wall_right) {
    const int64_t M = (int64_t)n * n * n;
    const int64_t nc = ncl + 4;
    double dv = 2.0 * L / n;
    double *sig = calloc((size_t)nc, sizeof(double));
    memcpy(out, field, sizeof(double) * nc * M);
    for (int64_t j = 0; j < M; ++j) {
        double v1 = dv * ((int)(j / (n * n)) - n / 2);
        for (int64_t c = 1; c <= ncl + 2; ++c) {
            double fm = field[(c - 1) * M + j], f0 = field[c * M + j], fp = field[(c + 1) * M + j];
            sig[c] = bo_minmod3((fp - f0) / (x_ext[c + 1] - x_ext[c]),
                                (f0 - fm) / (x_ext[c] - x_ext[c - 1]),
                                (fp - fm) / (x_ext[c + 1] - x_ext[c - 1]));
        }
        if (wall_left) { sig[1] = 0.0; sig[2] = 0.0; }
        if (wall_right) { sig[ncl + 2] = 0.0; sig[ncl + 1] = 0.0; }
        /* faces between c and c+1 for c = 1 .. ncl+1 */
        double Fprev = 0.0;
        for (int64_t c = 1; c <= ncl + 1; ++c) {
            double F;
            if (v1 >= 0.0) F = v1 * (field[c * M + j] + 0.5 * dx_ext[c] * sig[c]);
            else F = v1 * (field[(c + 1) * M + j] - 0.5 * dx_ext[c + 1] * sig[c + 1]);
            if (c >= 2) out[c * M + j] = field[c * M + j] - dt / dx_ext[c] * (F - Fprev);
            Fprev = F;
        }
    }
    free(sig);
}

/* plan_decomposition: contiguous ranges balanced to +-1,
 * larger ranges first.  Returns 0, or 2 if more ranks than cells. */
int bo_plan_decomposition(int64_t ncells, int nranks, int64_t *start, int64_t *count) {
    if (nranks < 1 || ncells < nranks) return 2;
    int64_t base = ncells / nranks, rem = ncells % nranks, s = 0;
    for (int r = 0; r < nranks; ++r) {
        int64_t c = base + (r < rem ? 1 : 0);
        start[r] = s;
        count[r] = c;
        s += c;
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* direct_collision_oracle: quadrature of the strong  */
/* form Q(f,f)(v) = sum_{v*} w* |u|^lambda b sum_sigma w_sigma          */
/*   [f(v') f(v*') - f(v) f(v*)],  b = 1/(4 pi),                        */
/* v', v*' = (v+v*)/2 +- |u| sigma / 2 (elastic collision rule),        */
/* sigma on S^2: Gauss-Legendre in cos(theta) x uniform azimuth,        */
/* f at off-lattice v', v*' by trilinear interpolation (0 off the       */
/* lattice).  Physics cross-check of the spectral operator; N <= 12.    */
/* ------------------------------------------------------------------ */
static double bo_trilinear(int n, double dv, const double *f, const double p[3]) {
    double g[3];
    int i0[3];
    double t[3];
    for (int a = 0; a < 3; ++a) {
        g[a] = p[a] / dv + n / 2;
        if (g[a] < 0.0 || g[a] > n - 1) return 0.0;
        i0[a] = (int)floor(g[a]);
        if (i0[a] >= n - 1) i0[a] = n - 2;
        t[a] = g[a] - i0[a];
    }
    double s = 0.0;
    for (int d = 0; d < 8; ++d) {
        int b1 = d >> 2 & 1, b2 = d >> 1 & 1, b3 = d & 1;
        double w = (b1 ? t[0] : 1 - t[0]) * (b2 ? t[1] : 1 - t[1]) * (b3 ? t[2] : 1 - t[2]);
        if (w == 0.0) continue;
        s += w * f[((int64_t)(i0[0] + b1) * n + (i0[1] + b2)) * n + (i0[2] + b3)];
    }
    return s;
}

/* returns 0, or 2 if n > 12 */
int bo_direct_collision(int n, double L, double lambda, const double *f, int n_theta, int n_phi, double *q,
                        int nthreads) {
    if (n > 12 || n_theta < 1 || n_phi < 1) return 2;
    const int64_t M = (int64_t)n * n * n;
    const double dv = 2.0 * L / n;
    double *gx = malloc(sizeof(double) * n_theta), *gw = malloc(sizeof(double) * n_theta);
    bo_gauss_legendre(n_theta, gx, gw);
    const int ns = n_theta * n_phi;
    double *sig = malloc(sizeof(double) * 3 * ns), *sw = malloc(sizeof(double) * ns);
    for (int k = 0; k < n_theta; ++k)
        for (int j = 0; j < n_phi; ++j) {
            double ct = gx[k], st = sqrt(fmax(0.0, 1.0 - ct * ct)), ph = 2.0 * BO_PI * j / n_phi;
            int s = k * n_phi + j;
            sig[3 * s] = st * cos(ph);
            sig[3 * s + 1] = st * sin(ph);
            sig[3 * s + 2] = ct;
            sw[s] = gw[k] * 2.0 * BO_PI / n_phi / (4.0 * BO_PI); /* b = 1/(4 pi) folded in */
        }
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 4)
#endif
    for (int64_t i = 0; i < M; ++i) {
        int i1 = (int)(i / (n * n)), i2 = (int)((i / n) % n), i3 = (int)(i % n);
        double v[3] = {dv * (i1 - n / 2), dv * (i2 - n / 2), dv * (i3 - n / 2)};
        double acc = 0.0;
        for (int64_t j = 0; j < M; ++j) {
            int j1 = (int)(j / (n * n)), j2 = (int)((j / n) % n), j3 = (int)(j % n);
            double vs[3] = {dv * (j1 - n / 2), dv * (j2 - n / 2), dv * (j3 - n / 2)};
            double u[3] = {v[0] - vs[0], v[1] - vs[1], v[2] - vs[2]};
            double um = sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
            if (um == 0.0) continue;
            double ws = axc(n, j1) * axc(n, j2) * axc(n, j3) * dv * dv * dv * pow(um, lambda);
            double c[3] = {0.5 * (v[0] + vs[0]), 0.5 * (v[1] + vs[1]), 0.5 * (v[2] + vs[2])};
            double gain = 0.0;
            for (int s = 0; s < ns; ++s) {
                double vp[3], vq[3];
                for (int a = 0; a < 3; ++a) {
                    vp[a] = c[a] + 0.5 * um * sig[3 * s + a];
                    vq[a] = c[a] - 0.5 * um * sig[3 * s + a];
                }
                double fp = bo_trilinear(n, dv, f, vp);
                if (fp == 0.0) continue;
                gain += sw[s] * fp * bo_trilinear(n, dv, f, vq);
            }
            acc += ws * (gain - f[i] * f[j]); /* sum_sigma sw = 1 */
        }
        q[i] = acc;
    }
    free(gx);
    free(gw);
    free(sig);
    free(sw);
    return 0;
}
