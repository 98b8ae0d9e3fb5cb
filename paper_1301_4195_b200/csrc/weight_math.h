// weight_math.h -- the convolution weight Ĝ(ξ,ζ), shared
// verbatim by the host table generator (host_weights.cpp, g++) and the
// on-device table generator (gen.cuh, nvcc) so both produce the same numbers.
//
//   Ĝ(ξ,ζ) = 4π/(2π)^{3/2} ∫_0^{r0} r^{λ+2} [sinc(a r) sinc(b r) − sinc(c r)] dr
//   a = β|ζ|/2, b = |ξ − βζ/2|, c = |ξ|
//
// λ ∈ {0,1}: the closed forms of PAPER.md:181-185 with p = a−b, q = a+b
// (SPEC.md:120,152), through the stable kernels
//   h(x)  = (x sin x + cos x − 1)/x²          = ∫_0^1 t cos(xt) dt
//   j1(x) = ((2−x²)cos x + 2x sin x − 2)/x⁴    = ∫_0^1 t³ sinc(xt) dt
//   j0(x) = (sin x − x cos x)/x³               = ∫_0^1 t² sinc(xt) dt
// (Taylor series near 0), every removable singularity (ζ=0, b=0, ξ=0, p=0)
// replaced by its limit, and p formed as (a²−b²)/(a+b) from the lattice's
// dot products so an exact a=b gives p=0 rather than a rounding residue -- the
// failure mode of the printed formula.
// Other λ: composite 16-point Gauss–Legendre panels.
#pragma once
#include <math.h>

#if defined(__CUDACC__)
#define BOLTZ_HD __host__ __device__ inline
#else
#define BOLTZ_HD inline
#endif

namespace boltz_w {

// sum_{n>=0} (-1)^n x^{2n} / ((2n + fact_shift)! * (2n + den0))
BOLTZ_HD double alt_series(double x2, int fact_shift, double den0) {
    double term = 1.0, s = 0.0;
    for (int n = 0; n < 30; ++n) {
        s += term / (2.0 * n + den0);
        term *= -x2 / ((2.0 * n + 1.0 + fact_shift) * (2.0 * n + 2.0 + fact_shift));
    }
    return s;
}
BOLTZ_HD double kern_h(double x) {
    if (fabs(x) < 1.0) return alt_series(x * x, 0, 2.0);
    return (x * sin(x) + cos(x) - 1.0) / (x * x);
}
BOLTZ_HD double kern_j1(double x) {
    if (fabs(x) < 1.5) return alt_series(x * x, 1, 4.0);
    const double x2 = x * x;
    return ((2.0 - x2) * cos(x) + 2.0 * x * sin(x) - 2.0) / (x2 * x2);
}
BOLTZ_HD double kern_j0(double x) {
    if (fabs(x) < 1.0) return alt_series(x * x, 1, 3.0);
    return (sin(x) - x * cos(x)) / (x * x * x);
}
BOLTZ_HD double kern_sinc(double x) {
    if (fabs(x) < 1e-3) {
        const double x2 = x * x;
        return 1.0 - x2 / 6.0 * (1.0 - x2 / 20.0 * (1.0 - x2 / 42.0));
    }
    return sin(x) / x;
}
BOLTZ_HD double prefactor() { return 4.0 * 3.14159265358979323846264338327950288 / pow(2.0 * 3.14159265358979323846264338327950288, 1.5); }

// closed form from |ζ|², |ξ|², ξ·ζ (all exact on the lattice)
BOLTZ_HD double closed_form(double lambda, double beta, double r0, double zz, double xx, double xz) {
    const double bb = xx - beta * xz + 0.25 * beta * beta * zz;
    const double a = 0.5 * beta * sqrt(zz), b = sqrt(bb > 0 ? bb : 0.0), c = sqrt(xx);
    double T1, T2;
    if (lambda == 1.0) {
        const double r2 = r0 * r0, r4 = r2 * r2;
        if (a == 0.0 && b == 0.0) T1 = 0.25 * r4;
        else if (a == 0.0) T1 = r4 * kern_j1(b * r0);
        else if (b == 0.0) T1 = r4 * kern_j1(a * r0);
        else {
            const double p = (beta * xz - xx) / (a + b), q = a + b;
            T1 = r2 * (kern_h(p * r0) - kern_h(q * r0)) / (2.0 * a * b);
        }
        T2 = r4 * kern_j1(c * r0);
    } else {
        const double r3 = r0 * r0 * r0;
        if (a == 0.0 && b == 0.0) T1 = r3 / 3.0;
        else if (a == 0.0) T1 = r3 * kern_j0(b * r0);
        else if (b == 0.0) T1 = r3 * kern_j0(a * r0);
        else {
            const double p = (beta * xz - xx) / (a + b), q = a + b;
            T1 = r0 * (kern_sinc(p * r0) - kern_sinc(q * r0)) / (2.0 * a * b);
        }
        T2 = r3 * kern_j0(c * r0);
    }
    return prefactor() * (T1 - T2);
}

// 16-point Gauss-Legendre nodes/weights on [-1,1]
struct Gauss16 {
    double x[16], w[16];
};
inline Gauss16 gauss16() {
    Gauss16 g{};
    const int n = 16;
    for (int i = 0; i < n / 2; ++i) {
        double z = cos(3.14159265358979323846264338327950288 * (i + 0.75) / (n + 0.5)), pp = 0;
        for (int it = 0; it < 100; ++it) {
            double p1 = 1.0, p2 = 0.0;
            for (int j = 1; j <= n; ++j) {
                const double p3 = p2;
                p2 = p1;
                p1 = ((2.0 * j - 1.0) * z * p2 - (j - 1.0) * p3) / j;
            }
            pp = n * (z * p1 - p2) / (z * z - 1.0);
            const double z1 = z;
            z = z1 - p1 / pp;
            if (fabs(z - z1) < 1e-16) break;
        }
        g.x[i] = -z;
        g.x[n - 1 - i] = z;
        g.w[i] = g.w[n - 1 - i] = 2.0 / ((1.0 - z * z) * pp * pp);
    }
    return g;
}

BOLTZ_HD double quadrature(double lambda, double beta, double r0, double zz, double xx, double xz, int panels,
                           const Gauss16& gl) {
    const double bb = xx - beta * xz + 0.25 * beta * beta * zz;
    const double a = 0.5 * beta * sqrt(zz), b = sqrt(bb > 0 ? bb : 0.0), c = sqrt(xx);
    const double h = r0 / panels;
    double s = 0.0;
    for (int p = 0; p < panels; ++p)
        for (int i = 0; i < 16; ++i) {
            const double r = p * h + 0.5 * h * (gl.x[i] + 1.0);
            s += 0.5 * h * gl.w[i] * pow(r, lambda + 2.0) * (kern_sinc(a * r) * kern_sinc(b * r) - kern_sinc(c * r));
        }
    return prefactor() * s;
}

// weight at lattice points: zeta = dz*k', xi = dz*m' with integer k', m'
BOLTZ_HD double lattice_weight(double lambda, double beta, double r0, int panels, const Gauss16& gl, double dz2,
                               int k1, int k2, int k3, int m1, int m2, int m3) {
    const double zz = dz2 * (double)(k1 * k1 + k2 * k2 + k3 * k3);
    const double xx = dz2 * (double)(m1 * m1 + m2 * m2 + m3 * m3);
    const double xz = dz2 * (double)(m1 * k1 + m2 * k2 + m3 * k3);
    return (lambda == 0.0 || lambda == 1.0) ? closed_form(lambda, beta, r0, zz, xx, xz)
                                            : quadrature(lambda, beta, r0, zz, xx, xz, panels, gl);
}

}  // namespace boltz_w
