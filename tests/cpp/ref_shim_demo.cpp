// The reference-typed drop-in on the GPU: the reference's own VelocityGrid
// (proj/src/velocity_grid.cpp, compiled in place), its UNMODIFIED
// boltz::SpectralTransform declaration (fourier.hpp:28-52) implemented by
// paper_1301_4195_b200/shim/fourier_cuda.cpp, the SPEC collision operations of
// shim/collision_cuda.hpp, and include/boltz_cuda.hpp in reference-error mode.
// Built by paper_1301_4195_b200/build.py:build_shim(); checked against the
// oracle by tests/test_reference_shim.py.
//
//   ref_shim_demo DIR N L LAMBDA
//     DIR/f.bin: ncells x N^3 doubles; DIR/G.bin: N^6 doubles (dense zeta-major)
//   writes DIR/fhat.bin (cell 0, complex), DIR/back.bin + DIR/max_imag.bin
//   (inverse of fhat), DIR/q.bin (collide of every cell), DIR/qhat.bin
//   (evaluate_qhat of cell 0's fhat), DIR/rk2.bin (one RK2 step, dt = 0.01),
//   and prints one line per error case it provokes and catches.
#include <complex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <limits>
#include <string>
#include <vector>

#include "boltz/errors.hpp"
#include "boltz/fourier.hpp"
#include "boltz/velocity_grid.hpp"
#include "boltz_cuda.hpp"
#include "collision_cuda.hpp"

template <typename T>
static std::vector<T> read_bin(const std::string& path) {
    std::ifstream f(path, std::ios::binary | std::ios::ate);
    if (!f) throw boltz::IoError("cannot read " + path);
    const std::streamsize n = f.tellg();
    std::vector<T> v(n / sizeof(T));
    f.seekg(0);
    f.read(reinterpret_cast<char*>(v.data()), n);
    return v;
}

template <typename T>
static void write_bin(const std::string& path, const std::vector<T>& v) {
    std::ofstream(path, std::ios::binary).write(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(T));
}

int main(int argc, char** argv) {
    if (argc != 5) {
        std::fprintf(stderr, "usage: ref_shim_demo DIR N L LAMBDA\n");
        return 2;
    }
    const std::string dir = argv[1];
    const int n = std::atoi(argv[2]);
    const double L = std::atof(argv[3]), lam = std::atof(argv[4]);
    try {
        const boltz::VelocityGrid grid = boltz::VelocityGrid::create(n, L);  // the reference's own code
        const size_t n3 = grid.size();
        const auto f = read_bin<double>(dir + "/f.bin");
        const auto G = read_bin<double>(dir + "/G.bin");

        // SpectralTransform, exactly as fourier.hpp declares it
        boltz::SpectralTransform st(grid);
        std::vector<std::complex<double>> fhat(n3);
        std::vector<double> back(n3);
        double mi = -1.0;
        st.forward(std::span<const double>(f.data(), n3), fhat);
        st.inverse(fhat, back, &mi);
        write_bin(dir + "/fhat.bin", fhat);
        write_bin(dir + "/back.bin", back);
        write_bin(dir + "/max_imag.bin", std::vector<double>{mi});

        // the SPEC collision operations, batched over every cell of f.bin
        boltz::CollisionGpu op(grid, boltz::GpuKernelSpec{lam, 1.0, 0.0}, G);
        std::vector<std::complex<double>> qhat(n3);
        boltz::evaluate_qhat(op, fhat, qhat);
        write_bin(dir + "/qhat.bin", qhat);
        std::vector<double> q(f.size());
        boltz::collide(op, f, q, 1.0);
        write_bin(dir + "/q.bin", q);
        std::vector<double> g = f;
        boltz::collision_rk2(op, g, 0.01);
        write_bin(dir + "/rk2.bin", g);

        // error cases: each must surface as the reference's own exception type
        std::vector<double> bad(f.begin(), f.begin() + n3);
        bad[17] = std::numeric_limits<double>::quiet_NaN();
        std::vector<double> qb(n3);
        try {
            boltz::collide(op, bad, qb, 1.0);
            std::printf("collide(NaN): no error\n");
        } catch (const boltz::NumericError& e) {
            std::printf("collide(NaN): NumericError category %d\n", static_cast<int>(e.category()));
        }
        try {
            boltz::collision_rk2(op, bad, 0.01);
            std::printf("collision_rk2(NaN): no error\n");
        } catch (const boltz::NumericError& e) {
            std::printf("collision_rk2(NaN): NumericError category %d\n", static_cast<int>(e.category()));
        }
        try {
            boltz::collide(op, std::span<const double>(f.data(), n3 - 1), std::span<double>(qb.data(), n3 - 1), 1.0);
            std::printf("collide(ragged): no error\n");
        } catch (const boltz::ConfigError& e) {
            std::printf("collide(ragged): ConfigError category %d\n", static_cast<int>(e.category()));
        }
        try {
            std::vector<std::complex<double>> small(n3 - 1);
            st.forward(std::span<const double>(f.data(), n3), small);
            std::printf("forward(short span): no error\n");
        } catch (const boltz::ConfigError& e) {
            std::printf("forward(short span): ConfigError category %d\n", static_cast<int>(e.category()));
        }
        try {
            const boltz::VelocityGrid g10 = boltz::VelocityGrid::create(10, L);  // valid grid, no compiled kernel
            boltz::SpectralTransform st10(g10);
            std::printf("SpectralTransform(N=10): no error\n");
        } catch (const boltz::ConfigError& e) {
            std::printf("SpectralTransform(N=10): ConfigError category %d\n", static_cast<int>(e.category()));
        }
        try {
            (void)boltz::VelocityGrid::create(5, L);  // the reference's own check (velocity_grid.cpp:12-13)
            std::printf("VelocityGrid(N=5): no error\n");
        } catch (const boltz::ConfigError& e) {
            std::printf("VelocityGrid(N=5): ConfigError category %d\n", static_cast<int>(e.category()));
        }
        // include/boltz_cuda.hpp in reference-error mode: a reference strang_step
        // that catches boltz::NumericError catches the wrapper's too
        try {
            boltz::cuda::CollisionOperator w(n, L, boltz::cuda::Kernel{lam, 1.0, 0.0}, G);
            std::vector<double> qw(n3);
            w.collide(bad, qw, 1.0);
            std::printf("cuda::CollisionOperator::collide(NaN): no error\n");
        } catch (const boltz::NumericError& e) {
            std::printf("cuda::CollisionOperator::collide(NaN): NumericError category %d\n",
                        static_cast<int>(e.category()));
        }
        std::printf("ref_shim_demo ok\n");
        return 0;
    } catch (const boltz::Error& e) {
        std::fprintf(stderr, "boltz::Error category %d: %s\n", static_cast<int>(e.category()), e.what());
        return static_cast<int>(e.category());
    }
}
