// host_weights.cpp -- the weight table Ĝ(ξ,ζ) on the host: the hot path's
// input as the reference produces it (generate_table / save_table /
// load_table), handed to boltz_create.  The math lives in
// weight_math.h, shared with the on-device generator (gen.cuh).
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
#include "weight_math.h"

namespace boltz_gpu {
void set_error(const std::string& s);
}

namespace {
constexpr double kPi = 3.14159265358979323846264338327950288;
const boltz_w::Gauss16& gl16() {
    static const boltz_w::Gauss16 g = boltz_w::gauss16();
    return g;
}
}  // namespace

extern "C" double boltz_weight(double lambda, double beta, double r0, const double xi[3], const double zeta[3],
                               int panels) {
    double zz = 0, xx = 0, xz = 0;
    for (int i = 0; i < 3; ++i) {
        zz += zeta[i] * zeta[i];
        xx += xi[i] * xi[i];
        xz += xi[i] * zeta[i];
    }
    if (lambda == 0.0 || lambda == 1.0) return boltz_w::closed_form(lambda, beta, r0, zz, xx, xz);
    return boltz_w::quadrature(lambda, beta, r0, zz, xx, xz, panels, gl16());
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
    if (!G) {
        boltz_gpu::set_error("generate_table: output is null");
        return BOLTZ_ERR_CONFIG;
    }
    const int64_t M = (int64_t)n * n * n;
    const double dz = kPi / L, dz2 = dz * dz;
    const int h = n / 2;
    const boltz_w::Gauss16& gl = gl16();
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
    for (int64_t k = 0; k < M; ++k) {
        const int k1 = (int)(k / (n * n)) - h, k2 = (int)((k / n) % n) - h, k3 = (int)(k % n) - h;
        double* Gk = G + k * M;
        for (int m1 = -h; m1 < h; ++m1)
            for (int m2 = -h; m2 < h; ++m2)
                for (int m3 = -h; m3 < h; ++m3)
                    *Gk++ = boltz_w::lattice_weight(lambda, beta, r0, panels, gl, dz2, k1, k2, k3, m1, m2, m3);
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
