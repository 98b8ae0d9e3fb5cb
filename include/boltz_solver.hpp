// boltz_solver.hpp -- header-only C++ host driver of the space-inhomogeneous
// problem over the C ABI (boltz_cuda.h): the reference's grid / time-stepping
// drivers in the reference's language, with every kernel on
// the GPU.  Mirrors paper_1301_4195_b200/solver.py (same call order, so the two
// produce bitwise-identical fields; tests/test_cpp_solver.py checks that).
//
//   strang_step(dt) = T(dt/2) o C_RK2(dt) o T(dt/2)
//   T(h):  SSP-RK2 of the FV step, ghost refresh before each
//          stage: halo exchange (NCCL / loopback) + physical ends; or the
//          SPEC's literal single stage f <- S(f) with one ghost refresh
//          (SPEC.md:342-345,471): TransportScheme::SingleStage
//   C_RK2: boltz_rk2_batch over the rank's interior cells (cell-local)
//
// Field: (ncl + 4) x N^3 doubles on the device, ghosts at 0,1 and ncl+2,ncl+3
// (SPEC.md:296).  Decomposition: contiguous ranges balanced to +-1
// (SPEC.md:426-444).  Build with nvcc, or g++ -I<cuda>/include -lcudart.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <cmath>
#include <cstdint>
#include <span>
#include <utility>
#include <vector>

#include "boltz_cuda.h"
#include "boltz_cuda.hpp"

namespace boltz::cuda {

inline void cuda_check(cudaError_t e) {
    if (e != cudaSuccess) throw_error(BOLTZ_ERR_CUDA, cudaGetErrorString(e));
}

// plan_decomposition: (start, count) per rank, contiguous,
// |count_r - count_s| <= 1, larger ranges first.
inline std::vector<std::pair<int64_t, int64_t>> plan_decomposition(int64_t ncells, int nranks) {
    if (nranks < 1 || ncells < nranks) throw_error(BOLTZ_ERR_CONFIG, "plan_decomposition: more ranks than cells");
    std::vector<std::pair<int64_t, int64_t>> out;
    const int64_t base = ncells / nranks, rem = ncells % nranks;
    int64_t s = 0;
    for (int r = 0; r < nranks; ++r) {
        const int64_t c = base + (r < rem ? 1 : 0);
        out.emplace_back(s, c);
        s += c;
    }
    return out;
}

// centres / widths of the global field with 2 mirrored ghost cells per end
// (ghost widths mirror the adjacent interior cells; scenarios.extend_ghosts)
inline void extend_ghosts(std::span<const double> x, std::span<const double> dx, std::vector<double>& xe,
                          std::vector<double>& dxe) {
    const size_t n = x.size();
    if (n < 2 || dx.size() != n) throw_error(BOLTZ_ERR_CONFIG, "extend_ghosts: need >= 2 cells");
    dxe.assign(n + 4, 0.0);
    dxe[0] = dx[1];
    dxe[1] = dx[0];
    for (size_t i = 0; i < n; ++i) dxe[i + 2] = dx[i];
    dxe[n + 2] = dx[n - 1];
    dxe[n + 3] = dx[n - 2];
    xe.assign(n + 4, 0.0);
    for (size_t i = 0; i < n; ++i) xe[i + 2] = x[i];
    xe[1] = x[0] - 0.5 * (dx[0] + dxe[1]);
    xe[0] = xe[1] - 0.5 * (dxe[1] + dxe[0]);
    xe[n + 2] = x[n - 1] + 0.5 * (dx[n - 1] + dxe[n + 2]);
    xe[n + 3] = xe[n + 2] + 0.5 * (dxe[n + 2] + dxe[n + 3]);
}

// physical end condition; WallBalanced is the
// flux-balanced wall extension (boltz_fill_boundary kind 2)
struct Boundary {
    enum Kind { Extrap = 0, Wall = 1, WallBalanced = 2 };
    Kind kind = Extrap;
    double Tw = 1.0;
    std::array<double, 3> Vw{0.0, 0.0, 0.0};
    bool is_wall() const { return kind != Extrap; }
};

// Device buffer (RAII)
template <typename T>
class DeviceArray {
public:
    DeviceArray() = default;
    explicit DeviceArray(size_t n) : n_(n) { cuda_check(cudaMalloc(&p_, n * sizeof(T))); }
    ~DeviceArray() {
        if (p_) cudaFree(p_);  // cudaFree(nullptr) is still illegal while a stream is capturing
    }
    DeviceArray(const DeviceArray&) = delete;
    DeviceArray& operator=(const DeviceArray&) = delete;
    DeviceArray(DeviceArray&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)) {}
    DeviceArray& operator=(DeviceArray&& o) noexcept {
        std::swap(p_, o.p_);
        std::swap(n_, o.n_);
        return *this;
    }
    void swap(DeviceArray& o) noexcept {
        std::swap(p_, o.p_);
        std::swap(n_, o.n_);
    }
    T* data() { return p_; }
    const T* data() const { return p_; }
    size_t size() const { return n_; }

private:
    T* p_ = nullptr;
    size_t n_ = 0;
};

// time integration of the transport sub-step T(h)
enum class TransportScheme {
    SspRk2 = 0,       // Heun: t1 = S(f), f <- f/2 + S(t1)/2 (DESIGN.md §5 item 4)
    SingleStage = 1,  // f <- S(f), one ghost refresh per sub-step
};

class Solver1D {
public:
    // x, dx: GLOBAL cell centres / widths; f0: this rank's interior cells,
    // ncl x N^3 host doubles (ncl from plan_decomposition(x.size(), world)).
    // halo: NCCL communicator for world > 1 (nullptr with the loopback driver).
    Solver1D(CollisionOperator& op, int n, double half_width, std::span<const double> x, std::span<const double> dx,
             std::span<const double> f0, int rank = 0, int world = 1, Boundary left = {}, Boundary right = {},
             double epsilon = 1.0, boltz_halo* halo = nullptr, cudaStream_t stream = nullptr,
             TransportScheme scheme = TransportScheme::SspRk2)
        : op_(op), n3_((int64_t)n * n * n), L_(half_width), rank_(rank), world_(world), left_(left), right_(right),
          eps_(epsilon), halo_(halo), s_(stream), scheme_(scheme) {
        cuda_check(cudaGetDevice(&device_));
        const auto plan = plan_decomposition((int64_t)x.size(), world);
        start_ = plan[rank].first;
        ncl_ = plan[rank].second;
        if (ncl_ < 2) throw_error(BOLTZ_ERR_CONFIG, "each rank needs at least 2 cells (2-cell halo, SPEC.md:438)");
        if ((int64_t)f0.size() != ncl_ * n3_) throw_error(BOLTZ_ERR_CONFIG, "f0 must hold this rank's ncl x N^3 values");
        std::vector<double> xe, dxe;
        extend_ghosts(x, dx, xe, dxe);
        dx_min_ = dx[0];
        for (double v : dx) dx_min_ = std::fmin(dx_min_, v);
        dx_host_.assign(dx.begin() + start_, dx.begin() + start_ + ncl_);
        x_ext_ = DeviceArray<double>(ncl_ + 4);
        dx_ext_ = DeviceArray<double>(ncl_ + 4);
        cuda_check(cudaMemcpy(x_ext_.data(), xe.data() + start_, (ncl_ + 4) * sizeof(double), cudaMemcpyHostToDevice));
        cuda_check(cudaMemcpy(dx_ext_.data(), dxe.data() + start_, (ncl_ + 4) * sizeof(double), cudaMemcpyHostToDevice));
        for (auto* b : {&field_, &tmp_, &tmp2_}) *b = DeviceArray<double>((ncl_ + 4) * n3_);
        cuda_check(cudaMemset(field_.data(), 0, (ncl_ + 4) * n3_ * sizeof(double)));
        cuda_check(cudaMemcpy(field_.data() + 2 * n3_, f0.data(), ncl_ * n3_ * sizeof(double), cudaMemcpyHostToDevice));
        red_ = DeviceArray<double>(8);
    }

    int64_t ncl() const { return ncl_; }
    int transport_stages() const { return scheme_ == TransportScheme::SingleStage ? 1 : 2; }
    int64_t cell_values() const { return n3_; }
    int64_t start() const { return start_; }
    double time() const { return t_; }
    double* field() { return field_.data(); }
    double* interior() { return field_.data() + 2 * n3_; }
    double cfl_dt(double cfl = 0.9) const { return cfl * dx_min_ / L_; }  // SPEC.md:379,408 (global min dx)

    // ghost refresh: halo exchange (unless exchange = false: the loopback driver
    // exchanged already) and the physical ends of the end ranks
    void fill_ghosts(bool exchange = true) {
        if (exchange && halo_) check(boltz_halo_exchange(halo_, field_.data(), ncl_, n3_, s_));
        fill_physical(field_.data());
    }

    // ghosts of the physical ends (wall / extrapolation) of `buf`, on the end ranks
    void fill_physical(double* buf) {
        if (rank_ == 0)
            check(boltz_fill_boundary(op_.handle(), buf, ncl_, x_ext_.data(), 0, left_.kind, left_.Tw,
                                      left_.Vw.data(), &sigma_w_[0], s_));
        if (rank_ == world_ - 1)
            check(boltz_fill_boundary(op_.handle(), buf, ncl_, x_ext_.data(), 1, right_.kind, right_.Tw,
                                      right_.Vw.data(), &sigma_w_[1], s_));
    }

    // ---- fused peer-memory halo (PeerGroup) ----
    // stage inputs / outputs BEFORE the stage runs (stage 1 rotates afterwards)
    double* stage_in(int stage) { return stage == 0 ? field_.data() : tmp_.data(); }
    double* stage_out(int stage) { return stage == 0 ? tmp_.data() : tmp2_.data(); }
    cudaStream_t stream() const { return s_; }
    int device() const { return device_; }
    boltz_ctx* op_handle() { return op_.handle(); }

    // one transport stage with the exchange fused into the kernel: the updated
    // edge cells go straight into the neighbours' stage outputs (left_dst /
    // right_dst); this rank's ghosts were written by its neighbours' previous op
    void transport_stage_peer(int stage, double h, double* left_dst, double* right_dst) {
        if (h * L_ > dx_min_ * (1 + 1e-12)) throw_error(BOLTZ_ERR_CONFIG, "transport: CFL violated (dt * L > min dx)");
        const int wl = rank_ == 0 && left_.is_wall(), wr = rank_ == world_ - 1 && right_.is_wall();
        double* in = stage_in(stage);
        fill_physical(in);
        check(boltz_transport_step_peer(op_.handle(), in, stage ? field_.data() : nullptr, stage ? 0.5 : 0.0,
                                        stage_out(stage), ncl_, x_ext_.data(), dx_ext_.data(), h, wl, wr, left_dst,
                                        right_dst, s_));
        if (scheme_ == TransportScheme::SingleStage) {
            field_.swap(tmp_);  // field = S(f)
        } else if (stage == 1) {
            field_.swap(tmp_);
            tmp2_.swap(field_);
        }
    }

    // the collision step + its half of the exchange: the post-collision edge
    // cells into the neighbours' fields' ghosts
    void collide_peer(double dt, double* left_dst, double* right_dst) {
        collide(dt);
        check(boltz_store_edges(op_.handle(), interior(), ncl_, left_dst, right_dst, s_));
    }

    // stage of the transport sub-step.  SSP-RK2: stage 0: t1 = S(f);
    // stage 1: f <- f/2 + S(t1)/2.  SingleStage: stage 0: f <- S(f).
    // S = one FV step after a ghost refresh of its input
    void transport_stage(int stage, double h, bool exchange = true) {
        const int wl = rank_ == 0 && left_.is_wall(), wr = rank_ == world_ - 1 && right_.is_wall();
        if (scheme_ == TransportScheme::SingleStage) {
            refresh_and_step(tmp_.data(), nullptr, 0.0, h, wl, wr, exchange);
            field_.swap(tmp_);  // field = S(f)
            return;
        }
        if (stage == 0) {
            refresh_and_step(tmp_.data(), nullptr, 0.0, h, wl, wr, exchange);
        } else {
            field_.swap(tmp_);  // field = t1, tmp = f^n
            refresh_and_step(tmp2_.data(), tmp_.data(), 0.5, h, wl, wr, exchange);
            tmp2_.swap(field_);  // field = out, tmp2 = t1
        }
    }

    // Halo/compute overlap (the NCCL halo, >= 6 cells per rank): each transport
    // stage runs the exchange on a side stream while the rows that read no ghost
    // ([4, ncl)) are updated, then the four edge rows -- bitwise the plain stage
    // (boltz_transport_step_range; paper_1301_4195_b200/solver.py overlap_halo).
    void set_overlap_halo(bool on) {
        overlap_ = on;
        if (on && !side_) {
            cuda_check(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
            cuda_check(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
            cuda_check(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
        }
    }

    // ghost refresh of the field, then out = [alpha base + (1 - alpha)] S(field)
    void refresh_and_step(double* out, const double* base, double alpha, double h, int wl, int wr, bool exchange) {
        if (!(exchange && overlap_ && halo_ && ncl_ >= 6)) {
            fill_ghosts(exchange);
            check(boltz_transport_step(op_.handle(), field_.data(), base, alpha, out, ncl_, x_ext_.data(),
                                       dx_ext_.data(), h, wl, wr, s_));
            return;
        }
        cuda_check(cudaEventRecord(ev_fork_, s_));
        cuda_check(cudaStreamWaitEvent(side_, ev_fork_, 0));
        check(boltz_halo_exchange(halo_, field_.data(), ncl_, n3_, side_));
        cuda_check(cudaEventRecord(ev_join_, side_));
        fill_physical(field_.data());  // the physical ends' ghost rows: disjoint from the exchanged ones
        auto rows = [&](int64_t b, int64_t e) {
            check(boltz_transport_step_range(op_.handle(), field_.data(), base, alpha, out, ncl_, x_ext_.data(),
                                             dx_ext_.data(), h, wl, wr, b, e, s_));
        };
        rows(4, ncl_);
        cuda_check(cudaStreamWaitEvent(s_, ev_join_, 0));
        rows(2, 4);
        rows(ncl_, ncl_ + 2);
    }

    // field of the loopback driver's stage-1 exchange (t1 lives in tmp until the stage swaps it in)
    double* stage_input(int stage) { return stage == 0 ? field_.data() : tmp_.data(); }

    void transport(double h) {
        if (h * L_ > dx_min_ * (1 + 1e-12)) throw_error(BOLTZ_ERR_CONFIG, "transport: CFL violated (dt * L > min dx)");
        for (int stage = 0; stage < transport_stages(); ++stage) transport_stage(stage, h);
    }

    void collide(double dt) { check(boltz_rk2_batch(op_.handle(), interior(), ncl_, dt, 1.0 / eps_, BOLTZ_MEM_DEVICE, s_)); }

    void strang_step(double dt) {
        transport(0.5 * dt);
        collide(dt);
        transport(0.5 * dt);
        t_ += dt;
    }
    void advance_time(double dt) { t_ += dt; }

    // compute_moments of the interior: ncl x 7 host doubles
    std::vector<double> moments() {
        DeviceArray<double> m(ncl_ * 7);
        check(boltz_moments_batch(op_.handle(), interior(), m.data(), ncl_, BOLTZ_MEM_DEVICE, s_));
        std::vector<double> h(ncl_ * 7);
        cuda_check(cudaMemcpyAsync(h.data(), m.data(), h.size() * sizeof(double), cudaMemcpyDeviceToHost, s_));
        cuda_check(cudaStreamSynchronize(s_));
        return h;
    }

    // global (mass, x-momentum, energy) = sum_j dx_j (rho, rho V1, rho e)_j over all ranks
    std::array<double, 3> ledger() {
        const auto m = moments();
        double tot[3] = {0, 0, 0};
        for (int64_t j = 0; j < ncl_; ++j) {
            tot[0] += m[j * 7 + 0] * dx_host_[j];
            tot[1] += m[j * 7 + 1] * dx_host_[j];
            tot[2] += m[j * 7 + 4] * dx_host_[j];
        }
        if (halo_ && world_ > 1) {
            cuda_check(cudaMemcpyAsync(red_.data(), tot, sizeof tot, cudaMemcpyHostToDevice, s_));
            check(boltz_halo_allreduce_sum(halo_, red_.data(), 3, s_));
            cuda_check(cudaMemcpyAsync(tot, red_.data(), sizeof tot, cudaMemcpyDeviceToHost, s_));
            cuda_check(cudaStreamSynchronize(s_));
        }
        return {tot[0], tot[1], tot[2]};
    }

    // interior cells -> host (ncl x N^3)
    void download(std::span<double> out) {
        if ((int64_t)out.size() != ncl_ * n3_) throw_error(BOLTZ_ERR_CONFIG, "download: size must be ncl x N^3");
        cuda_check(cudaMemcpyAsync(out.data(), interior(), out.size() * sizeof(double), cudaMemcpyDeviceToHost, s_));
        cuda_check(cudaStreamSynchronize(s_));
    }

    double sigma_w(int side) const { return sigma_w_[side]; }

    // `steps` Strang steps with the device queue kept full: one eager step (the
    // library allocates its workspace and sets kernel attributes lazily, which
    // cannot happen under capture), then capture() + advance(steps - 1).
    void run(double dt, int steps) {
        if (steps < 4 || !s_) {
            for (int i = 0; i < steps; ++i) strang_step(dt);
            return;
        }
        strang_step(dt);
        capture(dt);
        advance(steps - 1);
    }

    // CUDA-graph replay: capture three Strang steps of size
    // dt on the solver's stream (three steps bring the field / scratch rotation
    // back to its start), with the library in asynchronous mode.  Needs a
    // non-default stream and one eager step first (see run()).  The NCCL halo
    // is captured too when world > 1.  Does not advance the state.
    void capture(double dt) {
        if (!s_) throw_error(BOLTZ_ERR_CONFIG, "capture: the solver needs a non-default stream");
        const double* p0[3] = {field_.data(), tmp_.data(), tmp2_.data()};
        check(boltz_set_async(op_.handle(), 1));
        cudaGraph_t g = nullptr;
        cuda_check(cudaStreamBeginCapture(s_, cudaStreamCaptureModeThreadLocal));
        try {
            for (int i = 0; i < 3; ++i) {
                transport(0.5 * dt);
                collide(dt);
                transport(0.5 * dt);
            }
        } catch (...) {
            cudaStreamEndCapture(s_, &g);
            if (g) cudaGraphDestroy(g);
            boltz_set_async(op_.handle(), 0);
            throw;
        }
        cuda_check(cudaStreamEndCapture(s_, &g));
        check(boltz_set_async(op_.handle(), 0));
        if (field_.data() != p0[0] || tmp_.data() != p0[1] || tmp2_.data() != p0[2]) {
            cudaGraphDestroy(g);
            throw_error(BOLTZ_ERR_CONFIG, "capture: buffer rotation did not close after 3 steps");
        }
        if (exec_) cudaGraphExecDestroy(exec_);
        exec_ = nullptr;
        const cudaError_t e = cudaGraphInstantiate(&exec_, g, 0);
        cudaGraphDestroy(g);
        cuda_check(e);
        graph_dt_ = dt;
    }

    // `steps` Strang steps of the captured dt: graph replays + eager remainder;
    // numeric errors are reported once, at the end (boltz_sync)
    void advance(int steps) {
        if (!exec_) throw_error(BOLTZ_ERR_CONFIG, "advance: capture() first");
        check(boltz_set_async(op_.handle(), 1));
        try {
            for (int i = 0; i < steps / 3; ++i) {
                cuda_check(cudaGraphLaunch(exec_, s_));
                t_ += 3 * graph_dt_;
            }
            for (int i = 0; i < steps % 3; ++i) strang_step(graph_dt_);
            check(boltz_sync(op_.handle(), s_));
        } catch (...) {
            boltz_set_async(op_.handle(), 0);
            throw;
        }
        check(boltz_set_async(op_.handle(), 0));
    }

    ~Solver1D() {
        if (exec_) cudaGraphExecDestroy(exec_);
        if (side_) {
            cudaStreamDestroy(side_);
            cudaEventDestroy(ev_fork_);
            cudaEventDestroy(ev_join_);
        }
    }
    Solver1D(const Solver1D&) = delete;
    Solver1D& operator=(const Solver1D&) = delete;

private:
    CollisionOperator& op_;
    int64_t n3_;
    double L_;
    int rank_, world_;
    int device_ = 0;
    Boundary left_, right_;
    double eps_;
    boltz_halo* halo_;
    cudaStream_t s_;
    TransportScheme scheme_;
    int64_t start_ = 0, ncl_ = 0;
    double dx_min_ = 0, t_ = 0;
    double sigma_w_[2] = {0, 0};
    std::vector<double> dx_host_;
    DeviceArray<double> x_ext_, dx_ext_, field_, tmp_, tmp2_, red_;
    cudaGraphExec_t exec_ = nullptr;
    double graph_dt_ = 0;
    bool overlap_ = false;
    cudaStream_t side_ = nullptr;
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
};

// One process driving the ranks of a sharded domain in lockstep -- several
// GPUs of one box (peer access over NVLink / NVSwitch) or virtual ranks of one
// device -- with the halo exchange fused into the transport kernel: every
// transport stage stores its updated edge cells straight into the neighbours'
// stage outputs, and the collision step stores its edge cells into the
// neighbours' fields (boltz_transport_step_peer / boltz_store_edges), so no
// separate exchange runs at all.  Ordering is by CUDA events only: before op t
// a rank's stream waits for its neighbours' op t-1 (two events per rank, by
// op parity), which covers both the ghosts it reads (RAW) and the ghosts it
// writes next door (their readers finished, WAR).  Each rank needs its own
// CollisionOperator (workspace) and its own stream.
class PeerGroup {
public:
    explicit PeerGroup(std::vector<Solver1D*> ranks) : r_(std::move(ranks)) {
        if (r_.empty()) throw_error(BOLTZ_ERR_CONFIG, "PeerGroup: no ranks");
        ev_.resize(2 * r_.size());
        for (size_t i = 0; i < r_.size(); ++i) {
            if (!r_[i]->stream()) throw_error(BOLTZ_ERR_CONFIG, "PeerGroup: every rank needs its own stream");
            cuda_check(cudaSetDevice(r_[i]->device()));
            for (int p = 0; p < 2; ++p) cuda_check(cudaEventCreateWithFlags(&ev_[2 * i + p], cudaEventDisableTiming));
            for (int d : {-1, 1}) {  // peer access to the neighbours' devices
                const long j = (long)i + d;
                if (j < 0 || j >= (long)r_.size() || r_[j]->device() == r_[i]->device()) continue;
                const cudaError_t e = cudaDeviceEnablePeerAccess(r_[j]->device(), 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_check(e);
                cudaGetLastError();
            }
        }
        // the first op's ghosts: every rank's edge cells into its neighbours' fields
        op([](size_t, double*, double*) {}, Kind::Prime);
    }
    ~PeerGroup() {
        for (cudaEvent_t e : ev_) cudaEventDestroy(e);
    }
    PeerGroup(const PeerGroup&) = delete;
    PeerGroup& operator=(const PeerGroup&) = delete;

    void strang_step(double dt) {
        for (int half = 0; half < 2; ++half) {
            for (int stage = 0; stage < r_[0]->transport_stages(); ++stage)
                op([&](size_t i, double* l, double* r) { r_[i]->transport_stage_peer(stage, 0.5 * dt, l, r); },
                   stage == 0 ? Kind::Stage0 : Kind::Stage1);
            if (half == 0) op([&](size_t i, double* l, double* r) { r_[i]->collide_peer(dt, l, r); }, Kind::Collide);
        }
        for (auto* s : r_) s->advance_time(dt);
    }

private:
    enum class Kind { Prime, Stage0, Stage1, Collide };

    // destinations (from the neighbours' pointers before anyone rotates), then
    // per rank: wait for the neighbours' previous op, run, record
    template <typename F>
    void op(F&& run, Kind k) {
        const size_t R = r_.size();
        std::vector<double*> L(R, nullptr), Rt(R, nullptr);
        for (size_t i = 0; i < R; ++i) {
            auto target = [&](size_t j) {
                return (k == Kind::Stage0) ? r_[j]->stage_out(0) : (k == Kind::Stage1) ? r_[j]->stage_out(1)
                                                                                       : r_[j]->field();
            };
            if (i > 0) L[i] = target(i - 1) + (r_[i - 1]->ncl() + 2) * r_[i - 1]->cell_values();
            if (i + 1 < R) Rt[i] = target(i + 1);
        }
        const int prev = parity_ ^ 1;
        for (size_t i = 0; i < R; ++i) {
            cuda_check(cudaSetDevice(r_[i]->device()));
            if (started_) {
                if (i > 0) cuda_check(cudaStreamWaitEvent(r_[i]->stream(), ev_[2 * (i - 1) + prev], 0));
                if (i + 1 < R) cuda_check(cudaStreamWaitEvent(r_[i]->stream(), ev_[2 * (i + 1) + prev], 0));
            }
            if (k == Kind::Prime)
                check(boltz_store_edges(r_[i]->op_handle(), r_[i]->interior(), r_[i]->ncl(), L[i], Rt[i],
                                        r_[i]->stream()));
            else
                run(i, L[i], Rt[i]);
            cuda_check(cudaEventRecord(ev_[2 * i + parity_], r_[i]->stream()));
        }
        started_ = true;
        parity_ ^= 1;
    }

    std::vector<Solver1D*> r_;
    std::vector<cudaEvent_t> ev_;
    int parity_ = 0;
    bool started_ = false;
};

// One Strang step of n virtual ranks of one device (loopback backend,
// SPEC.md:470): the ghost exchange runs between per-rank fields before every
// transport stage; bitwise equal to one rank (tests/test_cpp_solver.py).
inline void strang_step_loopback(std::vector<Solver1D*>& ranks, double dt, cudaStream_t s = nullptr) {
    std::vector<double*> fields(ranks.size());
    std::vector<int64_t> ncl(ranks.size());
    for (size_t r = 0; r < ranks.size(); ++r) ncl[r] = ranks[r]->ncl();
    auto exchange = [&](int stage, int64_t cells) {
        for (size_t r = 0; r < ranks.size(); ++r) fields[r] = ranks[r]->stage_input(stage);
        check(boltz_halo_exchange_loopback(fields.data(), ncl.data(), (int)ranks.size(), cells, s));
    };
    for (int half = 0; half < 2; ++half) {
        for (int stage = 0; stage < ranks[0]->transport_stages(); ++stage) {
            exchange(stage, ranks[0]->cell_values());
            for (auto* r : ranks) r->transport_stage(stage, 0.5 * dt, false);
        }
        if (half == 0)
            for (auto* r : ranks) r->collide(dt);
    }
    for (auto* r : ranks) r->advance_time(dt);
}

}  // namespace boltz::cuda
