// C++ caller of the boundary through include/boltz_cuda.hpp: the way the
// reference's timestepper would drive the GPU collision step.  Built by
// tests/test_cpp_wrapper.py (compile on CPU, run on GPU).
#include <cmath>
#include <cstdio>
#include <vector>

#include "boltz_cuda.hpp"

int main() {
    const int n = 8;
    const double L = 5.0, dv = 2 * L / n;
    try {
        boltz::cuda::Kernel k;
        auto G = boltz::cuda::generate_table(n, L, k);
        boltz::cuda::CollisionOperator op(n, L, k, G);
        const size_t m = op.cell_size();
        std::vector<double> f(2 * m);
        for (int c = 0; c < 2; ++c)
            for (int i = 0; i < n; ++i)
                for (int j = 0; j < n; ++j)
                    for (int l = 0; l < n; ++l) {
                        double v1 = dv * (i - n / 2) - (c ? 0.7 : -0.7), v2 = dv * (j - n / 2), v3 = dv * (l - n / 2);
                        f[c * m + (i * n + j) * n + l] = std::exp(-(v1 * v1 + v2 * v2 + v3 * v3) / 2) / std::pow(2 * M_PI, 1.5);
                    }
        std::vector<double> q(2 * m);
        op.collide(f, q, 1.0);
        double mass = 0, qmax = 0;
        auto c = [&](int a) { return (a == 0 || a == n - 1) ? 0.5 : 1.0; };  // trapezoid (velocity_grid.cpp:25-27)
        for (size_t i = 0; i < m; ++i) {
            const int a = i / (n * n), b = (i / n) % n, d = i % n;
            mass += q[i] * c(a) * c(b) * c(d);
            qmax = std::fmax(qmax, std::fabs(q[i]));
        }
        op.collision_rk2(f, 0.01, 1.0);
        std::printf("collide ok: |sum Q| / max|Q| = %.3e\n", std::fabs(mass) / qmax);
        try {
            std::vector<double> bad(m + 1);
            op.collide(bad, bad, 1.0);
        } catch (const boltz::cuda::Error& e) {
            std::printf("config error category %d\n", boltz::cuda::category_of(e));
        }
        return 0;
    } catch (const boltz::cuda::Error& e) {
        std::printf("error category %d: %s\n", boltz::cuda::category_of(e), e.what());
        return boltz::cuda::category_of(e);
    }
}
