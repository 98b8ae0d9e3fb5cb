// ref_grid_driver.cpp -- TEST INFRASTRUCTURE (oracle pin).
// Links the reference's own VelocityGrid (/root/reference/proj/src/velocity_grid.cpp,
// compiled in place by oracle/Makefile, never copied) and prints, as JSON, the
// grid quantities SPEC.md:30-47 pins, plus the ConfigError categories of
// velocity_grid.cpp:12-15.  tests/golden/make_golden.py freezes the output.
#include <cstdio>
#include "boltz/errors.hpp"
#include "boltz/velocity_grid.hpp"

int main() {
    const int ns[] = {4, 6, 8, 16, 24, 32};
    const double Ls[] = {1.0, 5.0, 6.0, 8.0};
    std::printf("{\"grids\": [\n");
    bool first = true;
    for (int n : ns)
        for (double L : Ls) {
            auto g = boltz::VelocityGrid::create(n, L);
            std::printf("%s{\"n\": %d, \"L\": %.17g, \"dv\": %.17g, \"dzeta\": %.17g, \"v\": [",
                        first ? "" : ",\n", n, L, g.dv, g.dzeta);
            first = false;
            for (int k = 0; k < n; ++k) std::printf("%s%.17g", k ? ", " : "", g.v_nodes[k]);
            std::printf("], \"zeta\": [");
            for (int k = 0; k < n; ++k) std::printf("%s%.17g", k ? ", " : "", g.zeta_nodes[k]);
            std::printf("], \"coeff\": [");
            for (int k = 0; k < n; ++k) std::printf("%s%.17g", k ? ", " : "", g.axis_coeff[k]);
            std::printf("], \"vel_weight_corner\": %.17g, \"fourier_weight_center\": %.17g, \"flat_123\": %zu}",
                        g.vel_weight(0, 0, 0), g.fourier_weight(n / 2, n / 2, n / 2), g.flat(1, 2, 3));
        }
    std::printf("],\n\"errors\": [");
    struct { int n; double L; } bad[] = {{3, 1.0}, {2, 1.0}, {7, 5.0}, {8, 0.0}, {8, -1.0}};
    bool f2 = true;
    for (auto b : bad) {
        int cat = 0;
        try { boltz::VelocityGrid::create(b.n, b.L); } catch (const boltz::Error& e) { cat = static_cast<int>(e.category()); }
        std::printf("%s{\"n\": %d, \"L\": %.17g, \"category\": %d}", f2 ? "" : ", ", b.n, b.L, cat);
        f2 = false;
    }
    std::printf("]}\n");
    return 0;
}
