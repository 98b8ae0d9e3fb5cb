// The C++ host driver (include/boltz_solver.hpp) on the GPU: the reference's
// time-stepping loop in the reference's language over the C ABI.  Built and
// checked by tests/test_cpp_solver.py against the Python driver (solver.py).
//
//   solver_demo DIR N L LAMBDA TW DT STEPS NRANKS MODE [SCHEME]
//     SCHEME ssp (default): SSP-RK2 transport sub-steps; single: the SPEC's
//                    single-stage transport sub-step
//     DIR/x.bin, DIR/dx.bin: Nx doubles; DIR/f0.bin: Nx x N^3 doubles
//     MODE nccl:     one rank, an NCCL communicator of world 1 (exchange is
//                    then a no-op; allreduce of the ledger is exercised)
//     MODE nccl_overlap: the same with the halo/compute overlap (side stream,
//                    split transport rows) and CUDA-graph replay
//     MODE loopback: NRANKS virtual ranks of one device
//     MODE peer:     NRANKS ranks of one device, each with its own context and
//                    stream, halo fused into the transport kernels (PeerGroup)
//     MODE graph:    one rank on its own stream: one eager step, then 3 Strang
//                    steps captured in a CUDA graph and replayed (Solver1D::run)
//   writes DIR/out_<MODE>_<NRANKS>.bin (Nx x N^3) and prints the ledger.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <memory>
#include <string>
#include <vector>

#include "boltz_solver.hpp"

using namespace boltz::cuda;

static std::vector<double> read_bin(const std::string& path) {
    std::ifstream f(path, std::ios::binary | std::ios::ate);
    if (!f) throw_error(BOLTZ_ERR_IO, "cannot read " + path);
    const std::streamsize n = f.tellg();
    std::vector<double> v(n / sizeof(double));
    f.seekg(0);
    f.read(reinterpret_cast<char*>(v.data()), n);
    return v;
}

int main(int argc, char** argv) {
    if (argc != 10 && argc != 11) {
        std::fprintf(stderr, "usage: solver_demo DIR N L LAMBDA TW DT STEPS NRANKS MODE [SCHEME]\n");
        return 2;
    }
    const std::string dir = argv[1], mode = argv[9], scheme_name = argc == 11 ? argv[10] : "ssp";
    const TransportScheme scheme = scheme_name == "single" ? TransportScheme::SingleStage : TransportScheme::SspRk2;
    const int n = std::atoi(argv[2]), steps = std::atoi(argv[7]), nranks = std::atoi(argv[8]);
    const double L = std::atof(argv[3]), lam = std::atof(argv[4]), Tw = std::atof(argv[5]), dt = std::atof(argv[6]);
    try {
        const auto x = read_bin(dir + "/x.bin"), dx = read_bin(dir + "/dx.bin"), f0 = read_bin(dir + "/f0.bin");
        const size_t nx = x.size(), n3 = (size_t)n * n * n;
        Kernel k;
        k.lambda = lam;
        CollisionOperator op(n, L, k, CollisionOperator::Generated{});
        Boundary left{Boundary::Wall, Tw}, right{Boundary::Extrap, 1.0};
        std::vector<double> out(nx * n3);
        std::array<double, 3> led0{}, led1{};
        if (mode == "nccl" || mode == "nccl_overlap") {
            unsigned char id[BOLTZ_HALO_ID_BYTES];
            check(boltz_halo_unique_id(id));
            boltz_halo* halo = nullptr;
            check(boltz_halo_create(0, 1, id, 0, &halo));
            cudaStream_t st = nullptr;  // graph replay needs a non-default stream
            if (mode == "nccl_overlap") cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            {
                Solver1D s(op, n, L, x, dx, f0, 0, 1, left, right, 1.0, halo, st, scheme);
                led0 = s.ledger();
                if (mode == "nccl_overlap") {  // halo on a side stream beside the ghost-free rows, graph replay
                    s.set_overlap_halo(true);
                    s.run(dt, steps);
                } else {
                    for (int i = 0; i < steps; ++i) s.strang_step(dt);
                }
                led1 = s.ledger();
                s.download(out);
                // the ledger all-reduce of a world-1 communicator is the identity
                DeviceArray<double> buf(3);
                cuda_check(cudaMemset(buf.data(), 0, 3 * sizeof(double)));
                check(boltz_halo_allreduce_sum(halo, buf.data(), 3, nullptr));
                cuda_check(cudaDeviceSynchronize());
            }
            if (st) cuda_check(cudaStreamDestroy(st));
            check(boltz_halo_destroy(halo));
        } else if (mode == "peer") {
            const auto plan = plan_decomposition((int64_t)nx, nranks);
            std::vector<std::unique_ptr<CollisionOperator>> ops;
            std::vector<std::unique_ptr<Solver1D>> ranks;
            std::vector<cudaStream_t> streams(nranks);
            std::vector<Solver1D*> ptrs;
            for (int r = 0; r < nranks; ++r) {
                cuda_check(cudaStreamCreateWithFlags(&streams[r], cudaStreamNonBlocking));
                ops.push_back(std::make_unique<CollisionOperator>(n, L, k, CollisionOperator::Generated{}));
                std::span<const double> f0r(f0.data() + plan[r].first * n3, plan[r].second * n3);
                ranks.push_back(std::make_unique<Solver1D>(*ops.back(), n, L, x, dx, f0r, r, nranks, left, right, 1.0,
                                                           nullptr, streams[r], scheme));
                ptrs.push_back(ranks.back().get());
            }
            {
                PeerGroup group(ptrs);
                for (int i = 0; i < steps; ++i) group.strang_step(dt);
            }
            for (int r = 0; r < nranks; ++r)
                ptrs[r]->download(std::span<double>(out.data() + plan[r].first * n3, plan[r].second * n3));
            ranks.clear();
            ops.clear();
            for (auto st : streams) cuda_check(cudaStreamDestroy(st));
        } else if (mode == "graph") {
            cudaStream_t st;
            cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            {
                Solver1D s(op, n, L, x, dx, f0, 0, 1, left, right, 1.0, nullptr, st, scheme);
                led0 = s.ledger();
                s.run(dt, steps);
                led1 = s.ledger();
                s.download(out);
            }
            cuda_check(cudaStreamDestroy(st));
        } else {
            const auto plan = plan_decomposition((int64_t)nx, nranks);
            std::vector<std::unique_ptr<Solver1D>> ranks;
            std::vector<Solver1D*> ptrs;
            for (int r = 0; r < nranks; ++r) {
                std::span<const double> f0r(f0.data() + plan[r].first * n3, plan[r].second * n3);
                ranks.push_back(std::make_unique<Solver1D>(op, n, L, x, dx, f0r, r, nranks, left, right, 1.0, nullptr,
                                                           nullptr, scheme));
                ptrs.push_back(ranks.back().get());
            }
            for (auto* r : ptrs) {
                const auto l = r->ledger();
                for (int a = 0; a < 3; ++a) led0[a] += l[a];
            }
            for (int i = 0; i < steps; ++i) strang_step_loopback(ptrs, dt);
            for (int r = 0; r < nranks; ++r) {
                const auto l = ptrs[r]->ledger();
                for (int a = 0; a < 3; ++a) led1[a] += l[a];
                ptrs[r]->download(std::span<double>(out.data() + plan[r].first * n3, plan[r].second * n3));
            }
        }
        const std::string path =
            dir + "/out_" + mode + "_" + std::to_string(nranks) + (argc == 11 ? "_" + scheme_name : "") + ".bin";
        std::ofstream(path, std::ios::binary).write(reinterpret_cast<const char*>(out.data()), out.size() * 8);
        std::printf("ledger mass %.17g -> %.17g\n", led0[0], led1[0]);
        return 0;
    } catch (const Error& e) {
        std::fprintf(stderr, "error category %d: %s\n", category_of(e), e.what());
        return category_of(e);
    }
}
