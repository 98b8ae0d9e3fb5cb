// host_weights.cpp -- the weight table Ĝ(ξ,ζ): the hot path's input, produced
// on the host and handed to boltz_create (SURVEY.md §2 "weights").
//
//   Ĝ(ξ,ζ) = 4π/(2π)^{3/2} ∫_0^{r0} r^{λ+2} [sinc(a r) sinc(b r) − sinc(c r)] dr
//   a = β|ζ|/2, b = |ξ − βζ/2|, c = |ξ|
//
// λ ∈ {0,1}: the closed forms of PAPER.md:181-185 with p = a−b, q = a+b
// (SPEC.md:120,152), evaluated through the stable kernels
//   h(x)  = (x sin x + cos x − 1)/x²          = ∫_0^1 t cos(xt) dt
//   j1(x) = ((2−x²)cos x + 2x sin x − 2)/x⁴    = ∫_0^1 t³ sinc(xt) dt
//   j0(x) = (sin x − x cos x)/x³               = ∫_0^1 t² sinc(xt) dt
// (Taylor series near 0), and every removable singularity (ζ=0, b=0, ξ=0, p=0)
// replaced by its limit.  p is formed as (a²−b²)/(a+b) from the lattice's
// integer dot products, so an exact a=b gives p=0 rather than a rounding
// residue -- the failure mode of the printed formula.
// Other λ: composite 16-point Gauss–Legendre panels.
// Layout: ζ-major, G[k][m].  Generation is a pure parallel map:
// bit-identical for any thread count.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../../include/boltz_cuda.h"

namespace {

constexpr double kPi = 3.14159265358979323846264338327950288;
const double kC0 = 4.0 * kPi / std::pow(2.0 * kPi, 1.5);

// sum_{n>=0} (-1)^n x^{2n} / ((2n + odd)! * (2n + den0))
inline double alt_series(double x2, int fact_shift, double den0) {
    // term_n = (-1)^n x^{2n} / (2n + fact_shift)!   (fact_shift 0 or 1)
    double term = 1.0, s = 0.0;
    for (int n = 0; n < 30; ++n) {
        s += term / (2.0 * n + den0);
        term *= -x2 / ((2.0 * n + 1.0 + fact_shift) * (2.0 * n + 2.0 + fact_shift));
    }
    return s;
}

inline double kern_h(double x) {
    if (std::fabs(x) < 1.0) return alt_series(x * x, 0, 2.0);
    return (x * std::sin(x) + std::cos(x) - 1.0) / (x * x);
}
inline double kern_j1(double x) {
    if (std::fabs(x) < 1.5) return alt_series(x * x, 1, 4.0);
    const double x2 = x * x;
    return ((2.0 - x2) * std::cos(x) + 2.0 * x * std::sin(x) - 2.0) / (x2 * x2);
}
inline double kern_j0(double x) {
    if (std::fabs(x) < 1.0) return alt_series(x * x, 1, 3.0);
    return (std::sin(x) - x * std::cos(x)) / (x * x * x);
}
inline double kern_sinc(double x) {
    if (std::fabs(x) < 1e-3) {
        const double x2 = x * x;
        return 1.0 - x2 / 6.0 * (1.0 - x2 / 20.0 * (1.0 - x2 / 42.0));
    }
    return std::sin(x) / x;
}

// closed form from the three squared norms and xi.zeta (all exact on the lattice)
double closed_form(double lambda, double beta, double r0, double zz, double xx, double xz) {
    const double bb = xx - beta * xz + 0.25 * beta * beta * zz;
    const double a = 0.5 * beta * std::sqrt(zz), b = std::sqrt(bb > 0 ? bb : 0.0), c = std::sqrt(xx);
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
    return kC0 * (T1 - T2);
}

struct Gauss16 {
    double x[16], w[16];
    Gauss16() {
        const int n = 16;
        for (int i = 0; i < n / 2; ++i) {
            double z = std::cos(kPi * (i + 0.75) / (n + 0.5)), pp = 0;
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
                if (std::fabs(z - z1) < 1e-16) break;
            }
            x[i] = -z;
            x[n - 1 - i] = z;
            w[i] = w[n - 1 - i] = 2.0 / ((1.0 - z * z) * pp * pp);
        }
    }
};

double quadrature(double lambda, double beta, double r0, double zz, double xx, double xz, int panels) {
    static const Gauss16 gl;
    const double bb = xx - beta * xz + 0.25 * beta * beta * zz;
    const double a = 0.5 * beta * std::sqrt(zz), b = std::sqrt(bb > 0 ? bb : 0.0), c = std::sqrt(xx);
    const double h = r0 / panels;
    double s = 0.0;
    for (int p = 0; p < panels; ++p)
        for (int i = 0; i < 16; ++i) {
            const double r = p * h + 0.5 * h * (gl.x[i] + 1.0);
            s += 0.5 * h * gl.w[i] * std::pow(r, lambda + 2.0) *
                 (kern_sinc(a * r) * kern_sinc(b * r) - kern_sinc(c * r));
        }
    return kC0 * s;
}

}  // namespace

namespace boltz_gpu {
void set_error(const std::string& s);
}

extern "C" double boltz_weight(double lambda, double beta, double r0, const double xi[3], const double zeta[3],
                               int panels) {
    double zz = 0, xx = 0, xz = 0;
    for (int i = 0; i < 3; ++i) {
        zz += zeta[i] * zeta[i];
        xx += xi[i] * xi[i];
        xz += xi[i] * zeta[i];
    }
    if (lambda == 0.0 || lambda == 1.0) return closed_form(lambda, beta, r0, zz, xx, xz);
    return quadrature(lambda, beta, r0, zz, xx, xz, panels);
}

extern "C" int boltz_generate_table(int n, double L, double lambda, double beta, double r0, int panels, double* G,
                                    int nthreads) {
    if (n < 4 || n % 2 != 0 || !(L > 0.0)) {
        boltz_gpu::set_error("generate_table: N must be even and >= 4 and L > 0");
        return BOLTZ_ERR_CONFIG;
    }
    if (!(lambda >= 0.0 && lambda <= 1.0) || !(r0 > 0.0) || !(beta > 0.0 && beta <= 1.0) || panels < 1) {
        boltz_gpu::set_error("generate_table: invalid kernel (0<=lambda<=1, 0<beta<=1, r0>0, panels>=1)");
        return BOLTZ_ERR_CONFIG;
    }
    const int64_t M = (int64_t)n * n * n;
    const double dz = kPi / L, dz2 = dz * dz;
    const int h = n / 2;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
    for (int64_t k = 0; k < M; ++k) {
        const int k1 = (int)(k / (n * n)) - h, k2 = (int)((k / n) % n) - h, k3 = (int)(k % n) - h;
        const double zz = dz2 * (double)(k1 * k1 + k2 * k2 + k3 * k3);
        double* Gk = G + k * M;
        for (int m1 = -h; m1 < h; ++m1)
            for (int m2 = -h; m2 < h; ++m2)
                for (int m3 = -h; m3 < h; ++m3) {
                    const double xx = dz2 * (double)(m1 * m1 + m2 * m2 + m3 * m3);
                    const double xz = dz2 * (double)(m1 * k1 + m2 * k2 + m3 * k3);
                    const double v = (lambda == 0.0 || lambda == 1.0)
                                         ? closed_form(lambda, beta, r0, zz, xx, xz)
                                         : quadrature(lambda, beta, r0, zz, xx, xz, panels);
                    *Gk++ = v;
                }
    }
    return BOLTZ_OK;
}

namespace {
struct TableHeader {
    char magic[8];
    uint32_t version;
    int32_t n;
    double L, lambda, beta, r0;
    int32_t panels;
    int32_t reserved;
};
static_assert(sizeof(TableHeader) == 56, "table header layout");
constexpr char kMagic[8] = {'B', 'O', 'L', 'T', 'Z', 'T', 'B', 'L'};
}  // namespace

extern "C" int boltz_save_table(const char* path, int n, double L, double lambda, double beta, double r0,
                                int panels, const double* G) {
    FILE* fp = std::fopen(path, "wb");
    if (!fp) {
        boltz_gpu::set_error(std::string("save_table: cannot open ") + path);
        return BOLTZ_ERR_IO;
    }
    TableHeader hd{};
    std::memcpy(hd.magic, kMagic, 8);
    hd.version = 1;
    hd.n = n;
    hd.L = L;
    hd.lambda = lambda;
    hd.beta = beta;
    hd.r0 = r0;
    hd.panels = panels;
    const size_t cnt = (size_t)n * n * n * n * n * n;
    bool ok = std::fwrite(&hd, sizeof hd, 1, fp) == 1 && std::fwrite(G, sizeof(double), cnt, fp) == cnt;
    ok = (std::fclose(fp) == 0) && ok;
    if (!ok) {
        boltz_gpu::set_error(std::string("save_table: write failed: ") + path);
        return BOLTZ_ERR_IO;
    }
    return BOLTZ_OK;
}

extern "C" int boltz_load_table(const char* path, int n, double L, double lambda, double beta, double r0,
                                int panels, double* G) {
    FILE* fp = std::fopen(path, "rb");
    if (!fp) {
        boltz_gpu::set_error(std::string("load_table: cannot open ") + path);
        return BOLTZ_ERR_IO;
    }
    TableHeader hd{};
    if (std::fread(&hd, sizeof hd, 1, fp) != 1 || std::memcmp(hd.magic, kMagic, 8) != 0 || hd.version != 1) {
        std::fclose(fp);
        boltz_gpu::set_error(std::string("load_table: corrupt header: ") + path);
        return BOLTZ_ERR_IO;
    }
    char buf[512];
    auto mismatch = [&](const char* what, double want, double got) {
        std::snprintf(buf, sizeof buf, "load_table: parameter mismatch: %s expected %.17g, file has %.17g", what,
                      want, got);
        boltz_gpu::set_error(buf);
        std::fclose(fp);
        return BOLTZ_ERR_CONFIG;
    };
    if (hd.n != n) return mismatch("N", n, hd.n);
    if (hd.L != L) return mismatch("L", L, hd.L);
    if (hd.lambda != lambda) return mismatch("lambda", lambda, hd.lambda);
    if (hd.beta != beta) return mismatch("beta", beta, hd.beta);
    if (hd.r0 != r0) return mismatch("r0", r0, hd.r0);
    if (hd.panels != panels) return mismatch("panels", panels, hd.panels);
    const size_t cnt = (size_t)n * n * n * n * n * n;
    std::vector<double> tmp(cnt);
    const size_t got = std::fread(tmp.data(), sizeof(double), cnt, fp);
    std::fclose(fp);
    if (got != cnt) {
        std::snprintf(buf, sizeof buf, "load_table: truncated payload: %zu of %zu values", got, cnt);
        boltz_gpu::set_error(buf);
        return BOLTZ_ERR_IO;
    }
    std::memcpy(G, tmp.data(), cnt * sizeof(double));
    return BOLTZ_OK;
}
