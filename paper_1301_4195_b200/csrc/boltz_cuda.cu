// boltz_cuda.cu -- context object and C ABI (include/boltz_cuda.h) of the
// B200 collision path.  Host orchestration only; the kernels live in
// transforms.cuh (K1/K3), conv.cuh (K2) and transport.cuh (K4).
#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <omp.h>
#include <string>
#include <vector>

#include "../../include/boltz_cuda.h"
#include "common.cuh"
#include "conv.cuh"
#include "fft.cuh"
#include "transforms.cuh"
#include "transport.cuh"
#include "probe.cuh"
#include "fused.cuh"
#include "line.cuh"
#include "gen.cuh"

#ifndef BOLTZ_LINE
#define BOLTZ_LINE 1  // K1 / K3 as one cell per CTA, one FFT line per thread (line.cuh) at N = 8, 16
#endif
#ifndef BOLTZ_FUSED
#define BOLTZ_FUSED 1  // single-kernel K1 / K3 when the N^3 cube fits in shared memory
#endif

namespace boltz_gpu {


thread_local std::string g_err;
void set_error(const std::string& s) { g_err = s; }

struct CudaError {
    std::string msg;
};

#define CK(call)                                                                                      \
    do {                                                                                              \
        cudaError_t e_ = (call);                                                                      \
        if (e_ != cudaSuccess)                                                                        \
            throw CudaError{std::string(#call) + ": " + cudaGetErrorString(e_) + " (" __FILE__ ":" + \
                            std::to_string(__LINE__) + ")"};                                          \
    } while (0)

static bool supported_n(int n) {
#define BOLTZ_SUP(N) if (n == N) return true;
    BOLTZ_FOR_EACH_N(BOLTZ_SUP)
#undef BOLTZ_SUP
    return false;
}

}  // namespace boltz_gpu

using namespace boltz_gpu;

// kernel classes for timing / launch counting
enum Kind : int { KIND_CONV = 0, KIND_FFT = 1, KIND_PROJECT = 2, KIND_LAYOUT = 3, KIND_TRANSPORT = 4, kKinds = 5 };

constexpr int kScheduleCell = 5;  // boltz_set_schedule: lane = output k3 (conv.cuh k_conv_cell), N <= 16
constexpr int kScheduleAuto = 6;  // boltz_set_schedule: chosen per call from the batch size (effective_schedule)

// A host thread that lives as long as its context and runs one job at a time.
// The bounce pipeline's feeder and drainer legs run on two of these instead of
// on per-call std::threads: thread start-up leaves the timed call, and libgomp
// keeps each leg's copy team (host_copy) alive from one call to the next.
struct JobThread {
    std::thread th;
    std::mutex m;
    std::condition_variable cv;
    std::function<void()> job;
    bool busy = false, stop = false;
    void start(std::function<void()> f) {
        std::unique_lock<std::mutex> lk(m);
        if (!th.joinable()) th = std::thread([this] { loop(); });
        job = std::move(f);
        busy = true;
        lk.unlock();
        cv.notify_all();
    }
    void wait() {
        std::unique_lock<std::mutex> lk(m);
        cv.wait(lk, [&] { return !busy; });
    }
    void loop() {
        std::unique_lock<std::mutex> lk(m);
        for (;;) {
            cv.wait(lk, [&] { return busy || stop; });
            if (stop) return;
            std::function<void()> f = std::move(job);
            lk.unlock();
            f();  // the legs catch their own errors (PipeSync::fail)
            lk.lock();
            busy = false;
            cv.notify_all();
        }
    }
    ~JobThread() {
        {
            std::lock_guard<std::mutex> g(m);
            stop = true;
        }
        cv.notify_all();
        if (th.joinable()) th.join();
    }
};

struct boltz_ctx {
    int n = 0;
    double L = 0, lambda = 0, beta = 0, r0 = 0;
    int device = 0;
    // folded convolution table (conv.cuh)
    double* dH = nullptr;
    int2* dEnt = nullptr;
    int* dRowStart = nullptr;
    int nent = 0, slab = 0;
    // Hermitian mirror schedule (conv.cuh k_conv_mirror) for collide / RK2
    bool mirror = false;
    bool mirror2 = false;  // k_conv_mirror2 (TMEM accumulators) instead of k_conv_mirror
    int64_t terms_plain = 0, terms_mirror = 0;  // executed K2 terms per cell eval (H table sizes)
    double* dMH = nullptr;
    int4* dMEnt = nullptr;
    int* dItems = nullptr;  // nitems x kItemInts, then the longest-first order
    int nitems = 0;
    int* dListK[3] = {nullptr, nullptr, nullptr};  // k_conv_kcsm (N = 24, 32): row lists of phases 0, 1, 2
    int nK[3] = {0, 0, 0};
    // workspace (group layout), capacity in cells (multiple of 32)
    int64_t cap = 0;
    double2* dA = nullptr;
    double2* dB = nullptr;
    double* dFs = nullptr;   // RK2 stage (user layout)
    // host-call pipeline: double-buffered staging (user layout, complex-sized) + copy streams
    int64_t stage_cap = 0;
    static constexpr int kMaxStageSlots = 4;
    // staging buffer pairs in flight (BOLTZ_STAGE_SLOTS, 2..4): with 3, the H2D of
    // chunk i+2 need not wait for chunk i's compute (cfg2 e2e 626k -> 640k evals/s)
    int stage_slots = 3;
    double* dStageIn[kMaxStageSlots] = {};
    double* dStageOut[kMaxStageSlots] = {};
    // pinned host bounce ring for PAGEABLE caller memory (run_host_pipelined):
    // the caller's chunk is memcpy'd by host threads into pinned memory while
    // the GPU works on the previous chunk, so the DMA keeps its pinned speed
    int64_t bounce_cap = 0;  // cells per slot
    double* hBounceIn[kMaxStageSlots] = {};
    double* hBounceOut[kMaxStageSlots] = {};
    double* hBounceMi[kMaxStageSlots] = {};
    static constexpr int kBounceBlocks = 16;  // D2H of a slot in up to 16 blocks, one event each
    cudaEvent_t ev_blk[kMaxStageSlots][kBounceBlocks] = {};
    JobThread feeder_thread, drainer_thread;  // the bounce pipeline's two host legs
    cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
    cudaEvent_t ev_h2d[kMaxStageSlots] = {}, ev_comp[kMaxStageSlots] = {}, ev_d2h[kMaxStageSlots] = {};
    // second compute stream + workspace: odd host-pipeline chunks run beside even
    // ones, so one chunk's last wave overlaps the next chunk's first
    cudaStream_t comp2 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    double2* dA2 = nullptr;
    double2* dB2 = nullptr;
    double* dFs2 = nullptr;
    unsigned long long* dMaxIm2 = nullptr;
    int64_t cap2 = 0;
    unsigned long long* dMaxIm = nullptr;
    int* dFlag = nullptr;
    int* hFlag = nullptr;    // pinned
    ProjConst pc{};
    int64_t table_bytes = 0, ws_bytes = 0;
    int panels = 64;  // Gauss-Legendre panels of the on-device generator (0 < lambda < 1)
    // per-kernel-class CUDA-event timing (bench.py roofline) and launch counts
    bool timing = false;
    bool async_mode = false;  // device-pointer calls return without a sync (boltz_set_async)
    int schedule = 0;         // K2: 0 throughput, 1..4 latency (segmented rows), 5 cell (boltz_set_schedule)
    int line_cpb = 2;         // cells per CTA of the line K1/K3 (1 inside the two-stream host pipeline)
    int num_sms = 148;        // of the context's device (grid-stride kernels)
    double2* dSeg = nullptr;  // latency schedule's segment partials
    int64_t seg_cap = 0;      // cells
    double2* dSeg2 = nullptr; // ... of the second workspace set (swap_workspace)
    int64_t seg_cap2 = 0;
    double2* dCell = nullptr; // cell schedule: contiguous f-hat cubes (k_cell_gather)
    int64_t cell_cap = 0;
    double2* dCell2 = nullptr;  // ... of the second workspace set
    int64_t cell_cap2 = 0;
    // once a call was captured into a CUDA graph, the graph holds the workspace
    // pointers: growing a buffer then retires the old one (freed at destroy)
    // instead of freeing it, so a later replay never touches freed memory
    bool graph_captured = false;
    std::vector<void*> retired;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<int> ev_kind;
    double ms[kKinds] = {0, 0, 0, 0, 0};
    int64_t launches[kKinds] = {0, 0, 0, 0, 0};
};

namespace {

int64_t n3_of(const boltz_ctx* c) { return (int64_t)c->n * c->n * c->n; }

// the dynamic shared-memory opt-in of kernel `fn` on `device`, once per (kernel, device)
// the group array X[g][idx][lane] (double2) as a 2D TMA tensor of doubles
// {2 kLanes, groups N^3}, rows 512 bytes apart; box = one i1 plane (N^2 rows)
// of cpb adjacent cells (line.cuh k_fwd_line_tma)
using TmapEncode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
TmapEncode tmap_encode() {  // the driver's cuTensorMapEncodeTiled, through the runtime (no -lcuda)
    static TmapEncode encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) throw CudaError{"cuTensorMapEncodeTiled unavailable"};
        return reinterpret_cast<TmapEncode>(fn);
    }();
    return encode;
}
CUtensorMap make_group_tmap(void* X, int64_t ngroups, int n3, int cpb) {
    const TmapEncode encode = tmap_encode();
    const int nn = (int)std::lround(std::cbrt((double)n3)) * (int)std::lround(std::cbrt((double)n3));
    CUtensorMap m;
    const cuuint64_t dim[2] = {2 * kLanes, (cuuint64_t)ngroups * n3};
    const cuuint64_t stride[1] = {2 * kLanes * sizeof(double)};
    const cuuint32_t box[2] = {(cuuint32_t)(2 * cpb), (cuuint32_t)nn};
    const cuuint32_t estride[2] = {1, 1};
    const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, X, dim, stride, box, estride,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError{"cuTensorMapEncodeTiled failed: " + std::to_string((int)r)};
    return m;
}

// a user array [cell][N^3] (double) as a 2D TMA tensor {N, cells N^2}: one row
// per line, box = one cell, 128-byte (N = 16) / 64-byte (N = 8) swizzle
// (line.cuh k_fwd_line_tma, swz<N>)
CUtensorMap make_cells_tmap(const double* f, int64_t ncells, int n) {
    CUtensorMap m;
    const cuuint64_t dim[2] = {(cuuint64_t)n, (cuuint64_t)ncells * n * n};
    const cuuint64_t stride[1] = {(cuuint64_t)n * sizeof(double)};
    const cuuint32_t box[2] = {(cuuint32_t)n, (cuuint32_t)(n * n)};
    const cuuint32_t estride[2] = {1, 1};
    const CUtensorMapSwizzle sw = n * 8 >= 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : n * 8 >= 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                                : CU_TENSOR_MAP_SWIZZLE_32B;
    const CUresult r = tmap_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(f), dim, stride,
                                     box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError{"cuTensorMapEncodeTiled (cells) failed: " + std::to_string((int)r)};
    return m;
}

void configure_smem(const void* fn, int device, int bytes) {
    static std::mutex m;
    static std::vector<std::pair<const void*, int>> done;
    std::lock_guard<std::mutex> g(m);
    for (const auto& d : done)
        if (d.first == fn && d.second == device) return;
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.emplace_back(fn, device);
}

// frees a workspace buffer, or retires it while a captured graph may use it
void release(boltz_ctx* c, void* p) {
    if (!p) return;
    if (c->graph_captured) c->retired.push_back(p);
    else cudaFree(p);
}

// The K2 schedule a batch of nc cells runs under.  kScheduleAuto picks it per
// call (B200, host-memory collide, us per call at N = 16, throughput / 4
// segments / 8 segments / cell: 1 cell 447 / 170 / 150 / 99, 4 cells 463 / 180 /
// 161 / 134, 8 cells 464 / 198 / 176 / 185, 64 cells 579 / 359 / 360 / 633;
// profiles/r2_small_host_calls.txt; 128 and 256 cells: solver.k2_schedule).
// The reference calls its operator one cell at a time, so the
// reference-typed shim runs under it.
int effective_schedule(const boltz_ctx* c, int64_t nc);

// marks the context's workspace as baked into a graph when `s` is capturing
int effective_schedule(const boltz_ctx* c, int64_t nc) {
    if (c->schedule != kScheduleAuto) return c->schedule;
    if (c->n > 16) return 0;
    if (nc <= 4) return kScheduleCell;
    if (nc <= 64) return 2;
    if (nc <= 256) return 1;
    return 0;
}

void note_capture(boltz_ctx* c, cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone) c->graph_captured = true;
}

// One-time kernel configuration (cudaFuncSetAttribute) PER DEVICE: the runtime
// keeps function attributes per device context, so one process driving several
// GPUs (PeerGroup, boltz_halo_create_all) must opt each device in.
struct PerDevice {
    std::mutex m;
    uint64_t mask = 0;
    template <class Fn>
    void once(int dev, Fn&& fn) {
        std::lock_guard<std::mutex> g(m);
        const uint64_t bit = 1ull << (dev & 63);
        if (mask & bit) return;
        fn();  // throws CudaError on failure; the bit stays clear
        mask |= bit;
    }
};

// Brackets one kernel launch with CUDA events on its stream when timing is on.
struct Timed {
    boltz_ctx* c;
    cudaStream_t s;
    Timed(boltz_ctx* c_, int kind, cudaStream_t s_) : c(c_), s(s_) {
        c->launches[kind]++;
        if (!c->timing) return;
        if (c->ev_used + 2 > c->ev_pool.size()) {
            for (int i = 0; i < 64; ++i) {
                cudaEvent_t e;
                CK(cudaEventCreate(&e));
                c->ev_pool.push_back(e);
            }
        }
        c->ev_kind.push_back(kind);
        CK(cudaEventRecord(c->ev_pool[c->ev_used], s));
    }
    ~Timed() {
        if (!c->timing) return;
        cudaEventRecord(c->ev_pool[c->ev_used + 1], s);
        c->ev_used += 2;
    }
};

// after a stream sync: fold the recorded event pairs into the per-kind totals
void collect_timing(boltz_ctx* c) {
    for (size_t i = 0; i < c->ev_kind.size(); ++i) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, c->ev_pool[2 * i], c->ev_pool[2 * i + 1]) == cudaSuccess)
            c->ms[c->ev_kind[i]] += ms;
    }
    c->ev_kind.clear();
    c->ev_used = 0;
}

void fill_twiddles() {
    std::vector<double2> tw(kTwTotal);
    const int ns[] = {4, 6, 8, 12, 16, 24, 32};
    for (int n : ns)
        for (int j = 0; j < n; ++j) {
            long double ang = -2.0L * 3.14159265358979323846264338327950288L * j / n;
            tw[tw_offset(n) + j] = make_double2((double)cosl(ang), (double)sinl(ang));
        }
    CK(cudaMemcpyToSymbol(c_tw, tw.data(), sizeof(double2) * kTwTotal));
}

// (C C^T)^{-1} for the projection; long double accumulation.
void build_projection(boltz_ctx* c) {
    const int n = c->n;
    const long double dv = 2.0L * c->L / n;
    long double A[5][5] = {};
    for (int i1 = 0; i1 < n; ++i1)
        for (int i2 = 0; i2 < n; ++i2)
            for (int i3 = 0; i3 < n; ++i3) {
                long double cc = (long double)axis_coeff(n, i1) * axis_coeff(n, i2) * axis_coeff(n, i3);
                long double w = cc * dv * dv * dv;
                long double v1 = dv * (i1 - n / 2), v2 = dv * (i2 - n / 2), v3 = dv * (i3 - n / 2);
                long double r[5] = {w, v1 * w, v2 * w, v3 * w, (v1 * v1 + v2 * v2 + v3 * v3) * w};
                for (int a = 0; a < 5; ++a)
                    for (int b = 0; b < 5; ++b) A[a][b] += r[a] * r[b];
            }
    // Gauss-Jordan inverse (SPD, well conditioned at these sizes)
    long double M[5][10] = {};
    for (int a = 0; a < 5; ++a) {
        for (int b = 0; b < 5; ++b) M[a][b] = A[a][b];
        M[a][5 + a] = 1.0L;
    }
    for (int col = 0; col < 5; ++col) {
        int piv = col;
        for (int r = col + 1; r < 5; ++r)
            if (fabsl(M[r][col]) > fabsl(M[piv][col])) piv = r;
        for (int k = 0; k < 10; ++k) std::swap(M[col][k], M[piv][k]);
        long double d = M[col][col];
        for (int k = 0; k < 10; ++k) M[col][k] /= d;
        for (int r = 0; r < 5; ++r)
            if (r != col) {
                long double f = M[r][col];
                for (int k = 0; k < 10; ++k) M[r][k] -= f * M[col][k];
            }
    }
    for (int a = 0; a < 5; ++a)
        for (int b = 0; b < 5; ++b) c->pc.ginv[a * 5 + b] = (double)M[a][5 + b];
    c->pc.dv = 2.0 * c->L / n;
    c->pc.half = n / 2;
}

// Is the caller's G mirror-symmetric, G(N-k, N-m) == G(k, m) for all k, m with
// every index >= 1, to 1e-14 of max|G|?  (True for the weights of SPEC.md:93-166,
// which depend on |zeta|, |xi|, |xi - beta zeta/2|; a table that is not keeps
// the plain schedule only.)
bool g_mirror_symmetric(int n, const double* G) {
    const int64_t n3 = (int64_t)n * n * n;
    double gmax = 0.0, dmax = 0.0;
#pragma omp parallel for reduction(max : gmax, dmax) schedule(static)
    for (int64_t k = 0; k < n3; ++k) {
        const int k1 = (int)(k / (n * n)), k2 = (int)((k / n) % n), k3 = (int)(k % n);
        if (!k1 || !k2 || !k3) continue;
        const int64_t km = ((int64_t)(n - k1) * n + (n - k2)) * n + (n - k3);
        for (int m1 = 1; m1 < n; ++m1)
            for (int m2 = 1; m2 < n; ++m2)
                for (int m3 = 1; m3 < n; ++m3) {
                    const int64_t m = ((int64_t)m1 * n + m2) * n + m3;
                    const int64_t mm = ((int64_t)(n - m1) * n + (n - m2)) * n + (n - m3);
                    const double a = G[k * n3 + m], b = G[km * n3 + mm];
                    gmax = std::max(gmax, std::fabs(a));
                    dmax = std::max(dmax, std::fabs(a - b));
                }
    }
    return dmax <= 1e-14 * gmax;
}

// Entries, their H offsets / band types and the slab term orders of one
// schedule (plain: every entry BT_FULL in the conv_rows / pipe_rows / kcs
// order; mirror: k_conv_mirror's typed single-tile bands).
struct TableLayout {
    std::vector<short2> term;
    TermSet ts{};
    std::vector<int4> entk;  // k1, k2, m1, m2
    std::vector<int2> meta;  // H offset, band type
    size_t hsize = 0;        // doubles
    bool partner_terms = false;  // terms flagged kMirrorTermFlag (k_conv_mirror2)
};

void layout_terms_plain(int n, TableLayout& T, int& slab) {
    const int t = conv_tile(n), nk = n / t;
    const int slab_kc = band_slab_kc(n, t);
    slab = nk * slab_kc;
    T.term.assign(slab, make_short2(-1, -1));  // slab term order (must match conv_rows)
    for (int kc = 0; kc < nk; ++kc) {
        int pos = kc * slab_kc;
        for (int ti = 0; ti < nk; ++ti) {
            const int sc = band_tile_sc(nk, kc, ti);
            for (int i = 0; i < n; ++i) {
                const int m3 = band_diag(n, nk, kc, ti, i);
                for (int kk = 0; kk < t; ++kk)
                    if (band_term(n, t, kc, sc, m3, kk)) T.term[pos++] = make_short2((short)(kc * t + kk), (short)m3);
            }
        }
    }
    T.ts.slab_max = slab;
    T.ts.slab[0] = slab;
}

void layout_terms_mirror(int n, TableLayout& T) {
    // slab of one typed band in band_tile order (band_diag(n, 1, 0, 0, i) == i;
    // kMirrorKS kk passes, pass-major), padded to even
    auto typed = [&](int ty) {
        std::vector<short2> v(band_slab_type(n, ty), make_short2(-1, -1));
        int pos = 0;
        for (int q = 0; q < kMirrorKS; ++q)
            for (int m3 = 0; m3 < n; ++m3)
                for (int kk = q * n / kMirrorKS; kk < (q + 1) * n / kMirrorKS; ++kk)
                    if (band_term_t(n, n, 0, 0, m3, kk, ty)) v[pos++] = make_short2((short)kk, (short)m3);
        return v;
    };
    const auto a = typed(BT_A), rest = typed(BT_REST);
    int off = 0;
    for (int ty = 0; ty < kBandTypes; ++ty) {
        std::vector<short2> v = ty == BT_A ? a : rest;
        if (ty == BT_FULL) v.insert(v.begin(), a.begin(), a.end());  // k_conv_mirror: A half, then REST half
        const int sl = mirror_slab(n, ty);
        if ((int)v.size() != sl) throw CudaError{"mirror slab layout mismatch"};
        T.ts.off[ty] = off;
        T.ts.slab[ty] = sl;
        T.ts.slab_max = std::max(T.ts.slab_max, sl);
        T.term.insert(T.term.end(), v.begin(), v.end());
        off += sl;
    }
}

// H values of every entry of a layout into dH, from the host G one k1-plane at
// a time (the dense N^6 table is never resident) or generated on the device.
void fill_table(boltz_ctx* c, const double* G_host, TableLayout& T, double* dH) {
    const int n = c->n;
    const int nent = (int)T.entk.size();
    std::vector<int> list(nent);
    for (int e = 0; e < nent; ++e) list[e] = e;
    std::stable_sort(list.begin(), list.end(), [&](int a, int b) { return T.entk[a].x < T.entk[b].x; });
    std::vector<int> kstart(n + 1, 0);
    for (int e = 0; e < nent; ++e) kstart[T.entk[e].x + 1]++;
    for (int k = 0; k < n; ++k) kstart[k + 1] += kstart[k];
    int4* dEntK = nullptr;
    int2* dMeta = nullptr;
    int* dList = nullptr;
    short2* dTerm = nullptr;
    double* dPlane = nullptr;
    const size_t n3 = (size_t)n * n * n, plane = (size_t)n * n * n3;
    try {
        CK(cudaMalloc(&dEntK, (size_t)nent * sizeof(int4)));
        CK(cudaMalloc(&dMeta, (size_t)nent * sizeof(int2)));
        CK(cudaMalloc(&dList, (size_t)nent * sizeof(int)));
        CK(cudaMalloc(&dTerm, T.term.size() * sizeof(short2)));
        CK(cudaMemcpy(dEntK, T.entk.data(), (size_t)nent * sizeof(int4), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dMeta, T.meta.data(), (size_t)nent * sizeof(int2), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dList, list.data(), (size_t)nent * sizeof(int), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dTerm, T.term.data(), T.term.size() * sizeof(short2), cudaMemcpyHostToDevice));
        TermSet ts = T.ts;
        ts.term = dTerm;
        const double dz = kPi / c->L, w3 = dz * dz * dz;
        if (!G_host) {  // on-device generation (gen.cuh)
            GenParams gp{};
            gp.lambda = c->lambda; gp.beta = c->beta; gp.r0 = c->r0; gp.dz2 = dz * dz; gp.w3 = w3;
            gp.panels = c->panels; gp.n = n; gp.gl = boltz_w::gauss16();
            const long long total = (long long)nent * ts.slab_max;
            k_gen_H<<<(unsigned)((total + 255) / 256), 256>>>(dH, dEntK, dMeta, nent, ts, gp);
            CK(cudaGetLastError());
        } else {
            CK(cudaMalloc(&dPlane, plane * sizeof(double)));
            for (int k1 = 0; k1 < n; ++k1) {
                const int e0 = kstart[k1], e1 = kstart[k1 + 1];
                const long long total = (long long)(e1 - e0) * ts.slab_max;
                // partner-row terms (k_conv_mirror2) of the entries of plane n - k1 need this plane
                const int kp = n - k1;
                const long long total_p = T.partner_terms && kp < n ? (long long)(kstart[kp + 1] - kstart[kp]) * ts.slab_max : 0;
                if (total == 0 && total_p == 0) continue;
                CK(cudaMemcpy(dPlane, G_host + (size_t)k1 * plane, plane * sizeof(double), cudaMemcpyHostToDevice));
                if (total_p) {
                    k_build_H<<<(unsigned)((total_p + 255) / 256), 256>>>(dPlane, dH, dEntK, dMeta, dList, kstart[kp],
                                                                          kstart[kp + 1], ts, n, w3, 1);
                    CK(cudaGetLastError());
                }
                if (total == 0) continue;
                k_build_H<<<(unsigned)((total + 255) / 256), 256>>>(dPlane, dH, dEntK, dMeta, dList, e0, e1, ts, n,
                                                                    w3, 0);
                CK(cudaGetLastError());
            }
        }
        CK(cudaDeviceSynchronize());
    } catch (...) {
        cudaFree(dEntK); cudaFree(dMeta); cudaFree(dList); cudaFree(dTerm); cudaFree(dPlane);
        throw;
    }
    cudaFree(dEntK); cudaFree(dMeta); cudaFree(dList); cudaFree(dTerm); cudaFree(dPlane);
}

// Plain schedule: output row (k1,k2) x representative input row (m1,m2); CSR
// row_start + the longest-first order (conv.cuh conv_row).
void build_table_plain(boltz_ctx* c, const double* G_host) {
    const int n = c->n, h = n / 2;
    TableLayout T;
    layout_terms_plain(n, T, c->slab);
    std::vector<int2> ent;
    std::vector<int> row_start(n * n + 1, 0);
    for (int k1 = 0; k1 < n; ++k1)
        for (int k2 = 0; k2 < n; ++k2) {
            row_start[k1 * n + k2] = (int)ent.size();
            for (int m1 = std::max(0, k1 - h + 1); m1 <= std::min(n - 1, k1 + h); ++m1)
                for (int m2 = std::max(0, k2 - h + 1); m2 <= std::min(n - 1, k2 + h); ++m2) {
                    const int s1 = k1 - m1 + h, s2 = k2 - m2 + h;
                    if (m1 < s1 || (m1 == s1 && m2 <= s2)) {
                        ent.push_back(make_int2((m1 * n + m2) * n, (s1 * n + s2) * n));
                        T.meta.push_back(make_int2((int)T.hsize, BT_FULL));
                        T.hsize += c->slab;
                        T.entk.push_back(make_int4(k1, k2, m1, m2));
                    }
                }
        }
    row_start[n * n] = (int)ent.size();
    c->nent = (int)ent.size();
    {   // processing order appended after the CSR offsets (conv.cuh conv_row): longest rows first
        std::vector<int> order(n * n);
        for (int r = 0; r < n * n; ++r) order[r] = r;
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
            return row_start[a + 1] - row_start[a] > row_start[b + 1] - row_start[b];
        });
        row_start.insert(row_start.end(), order.begin(), order.end());
        for (int r = 0; r < n * n; ++r) row_start.push_back(r);  // natural order
    }
    if (T.hsize >= (size_t)UINT32_MAX) throw CudaError{"weight table too large for 32-bit H offsets"};
    const size_t hbytes = T.hsize * sizeof(double);
    CK(cudaMalloc(&c->dH, hbytes));
    CK(cudaMalloc(&c->dEnt, ent.size() * sizeof(int2)));
    CK(cudaMalloc(&c->dRowStart, row_start.size() * sizeof(int)));
    CK(cudaMemcpy(c->dEnt, ent.data(), ent.size() * sizeof(int2), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->dRowStart, row_start.data(), row_start.size() * sizeof(int), cudaMemcpyHostToDevice));
    c->table_bytes += (int64_t)hbytes + (int64_t)ent.size() * 8 + (int64_t)row_start.size() * 4;
    c->terms_plain = (int64_t)T.hsize;
    fill_table(c, G_host, T, c->dH);
}

// Mirror schedule (conv.cuh k_conv_mirror): work items over rows / row pairs.
void build_table_mirror(boltz_ctx* c, const double* G_host) {
    const int n = c->n, h = n / 2;
    TableLayout T;
    layout_terms_mirror(n, T);
    std::vector<int4> ent;
    std::vector<int> items;
    std::vector<long long> cost;
    auto add = [&](int k1, int k2, int m1, int m2, int ty) {
        const int s1 = k1 - m1 + h, s2 = k2 - m2 + h;
        ent.push_back(make_int4((m1 * n + m2) * n, (s1 * n + s2) * n, (int)T.hsize, ty));
        T.meta.push_back(make_int2((int)T.hsize, ty));
        T.hsize += T.ts.slab[ty];
        T.entk.push_back(make_int4(k1, k2, m1, m2));
    };
    // representative input rows of output row (k1,k2) in the plain order, with
    // "interior" = all of m1, m2, s1, s2 in [2, N-2]
    auto reps = [&](int k1, int k2, auto&& fn) {
        for (int m1 = std::max(0, k1 - h + 1); m1 <= std::min(n - 1, k1 + h); ++m1)
            for (int m2 = std::max(0, k2 - h + 1); m2 <= std::min(n - 1, k2 + h); ++m2) {
                const int s1 = k1 - m1 + h, s2 = k2 - m2 + h;
                if (m1 < s1 || (m1 == s1 && m2 <= s2))
                    fn(m1, m2, mirror_interior(n, m1) && mirror_interior(n, m2) && mirror_interior(n, s1) &&
                                   mirror_interior(n, s2));
            }
    };
    for (int k1 = 0; k1 < n; ++k1)
        for (int k2 = 0; k2 < n; ++k2) {
            const int r = k1 * n + k2;
            const bool has = k1 >= 1 && k2 >= 1;
            const int rm = has ? (n - k1) * n + (n - k2) : -1;
            if (has && rm < r) continue;  // handled with its partner
            const bool pair = has && rm != r;
            const size_t first = ent.size();
            int it[kItemInts];
            it[0] = r;
            it[1] = pair ? rm : -1;
            it[2] = (int)ent.size();
            if (!pair) {
                reps(k1, k2, [&](int m1, int m2, bool) { add(k1, k2, m1, m2, BT_FULL); });
                it[3] = it[2];
                it[4] = it[5] = (int)ent.size();
            } else {
                const int j1 = n - k1, j2 = n - k2;
                reps(k1, k2, [&](int m1, int m2, bool in) { if (in) add(k1, k2, m1, m2, BT_A); });
                it[3] = (int)ent.size();
                reps(k1, k2, [&](int m1, int m2, bool in) { if (!in) add(k1, k2, m1, m2, BT_FULL); });
                reps(k1, k2, [&](int m1, int m2, bool in) { if (in) add(k1, k2, m1, m2, BT_REST); });
                it[4] = (int)ent.size();
                reps(j1, j2, [&](int m1, int m2, bool in) { if (!in) add(j1, j2, m1, m2, BT_FULL); });
                reps(j1, j2, [&](int m1, int m2, bool in) { if (in) add(j1, j2, m1, m2, BT_REST); });
                it[5] = (int)ent.size();
            }
            long long w = 0;
            for (size_t e = first; e < ent.size(); ++e) w += T.ts.slab[ent[e].w];
            cost.push_back(w);
            items.insert(items.end(), it, it + kItemInts);
        }
    c->nitems = (int)cost.size();
    {   // longest items first (the conv_row lpt order, per item)
        std::vector<int> order(c->nitems);
        for (int i = 0; i < c->nitems; ++i) order[i] = i;
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
        items.insert(items.end(), order.begin(), order.end());
    }
    if (T.hsize >= (size_t)INT32_MAX) throw CudaError{"mirror table too large for 32-bit H offsets"};
    const size_t hbytes = T.hsize * sizeof(double);
    CK(cudaMalloc(&c->dMH, hbytes));
    CK(cudaMalloc(&c->dMEnt, ent.size() * sizeof(int4)));
    CK(cudaMalloc(&c->dItems, items.size() * sizeof(int)));
    CK(cudaMemcpy(c->dMEnt, ent.data(), ent.size() * sizeof(int4), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->dItems, items.data(), items.size() * sizeof(int), cudaMemcpyHostToDevice));
    c->table_bytes += (int64_t)hbytes + (int64_t)ent.size() * 16 + (int64_t)items.size() * 4;
    c->terms_mirror = (int64_t)T.hsize;
    fill_table(c, G_host, T, c->dMH);
}

// Mirror schedule with TMEM accumulators (conv.cuh k_conv_mirror2): FULL slab
// [A band | REST band], I slab (type id BT_A) [A band | REST | REST' of the
// partner row, flagged].
void layout_terms_mirror2(int n, TableLayout& T) {
    std::vector<short2> a(m2_a(n), make_short2(-1, -1)), rest(m2_r(n), make_short2(-1, -1)), restp,
        rband(m2_r(n), make_short2(-1, -1));
    int pos = 0, rpos = 0;
    for (int m3 = 0; m3 < n; ++m3)  // band_tile order of the single-tile A and REST bands
        for (int kk = 0; kk < n; ++kk) {
            if (band_term_t(n, n, 0, 0, m3, kk, BT_A)) a[pos++] = make_short2((short)kk, (short)m3);
            if (band_term_t(n, n, 0, 0, m3, kk, BT_REST)) rband[rpos++] = make_short2((short)kk, (short)m3);
        }
    if (band_slab_type(n, BT_REST) != m2_r(n)) throw CudaError{"mirror2 REST piece size mismatch"};
    pos = 0;
    for (int k3 = 0; k3 < n; ++k3)  // m2_rest order
        for (int m3 = 0; m3 < n; ++m3)
            if (rest_term(n, k3, m3)) rest[pos++] = make_short2((short)k3, (short)m3);
    restp = rest;
    for (auto& t : restp)
        if (t.x >= 0) t.x = (short)(t.x + kMirrorTermFlag);
    T.term.clear();
    T.ts.off[BT_FULL] = 0;
    T.ts.slab[BT_FULL] = m2_slab(n, BT_FULL);
    T.term.insert(T.term.end(), a.begin(), a.end());
    T.term.insert(T.term.end(), rband.begin(), rband.end());
    T.ts.off[BT_A] = (int)T.term.size();
    T.ts.slab[BT_A] = m2_slab(n, BT_A);
    T.term.insert(T.term.end(), a.begin(), a.end());
    T.term.insert(T.term.end(), rest.begin(), rest.end());
    T.term.insert(T.term.end(), restp.begin(), restp.end());
    T.ts.off[BT_REST] = (int)T.term.size();
    T.ts.slab[BT_REST] = 0;
    T.ts.slab_max = m2_slab(n, BT_A);
    if ((int)T.term.size() != m2_slab(n, BT_FULL) + m2_slab(n, BT_A)) throw CudaError{"mirror2 slab layout mismatch"};
    T.partner_terms = true;
}

void build_table_mirror2(boltz_ctx* c, const double* G_host) {
    const int n = c->n, h = n / 2;
    TableLayout T;
    layout_terms_mirror2(n, T);
    std::vector<int4> ent;
    std::vector<int> items;
    std::vector<long long> cost;
    auto add = [&](int k1, int k2, int m1, int m2, int ty) {
        const int s1 = k1 - m1 + h, s2 = k2 - m2 + h;
        ent.push_back(make_int4((m1 * n + m2) * n, (s1 * n + s2) * n, (int)T.hsize, ty));
        T.meta.push_back(make_int2((int)T.hsize, ty));
        T.hsize += T.ts.slab[ty];
        T.entk.push_back(make_int4(k1, k2, m1, m2));
    };
    auto reps = [&](int k1, int k2, auto&& fn) {
        for (int m1 = std::max(0, k1 - h + 1); m1 <= std::min(n - 1, k1 + h); ++m1)
            for (int m2 = std::max(0, k2 - h + 1); m2 <= std::min(n - 1, k2 + h); ++m2) {
                const int s1 = k1 - m1 + h, s2 = k2 - m2 + h;
                if (m1 < s1 || (m1 == s1 && m2 <= s2))
                    fn(m1, m2, mirror_interior(n, m1) && mirror_interior(n, m2) && mirror_interior(n, s1) &&
                                   mirror_interior(n, s2));
            }
    };
    for (int k1 = 0; k1 < n; ++k1)
        for (int k2 = 0; k2 < n; ++k2) {
            const int r = k1 * n + k2;
            const bool has = k1 >= 1 && k2 >= 1;
            const int rm = has ? (n - k1) * n + (n - k2) : -1;
            if (has && rm < r) continue;  // handled with its partner
            const bool pair = has && rm != r;
            const size_t first = ent.size();
            int it[kItemInts];
            it[0] = r;
            it[1] = pair ? rm : -1;
            it[2] = (int)ent.size();
            if (!pair) {
                reps(k1, k2, [&](int m1, int m2, bool) { add(k1, k2, m1, m2, BT_FULL); });
                it[3] = it[2];
                it[4] = it[5] = (int)ent.size();
            } else {
                reps(k1, k2, [&](int m1, int m2, bool in) { if (in) add(k1, k2, m1, m2, BT_A); });
                it[3] = (int)ent.size();
                reps(k1, k2, [&](int m1, int m2, bool in) { if (!in) add(k1, k2, m1, m2, BT_FULL); });
                it[4] = (int)ent.size();
                reps(n - k1, n - k2, [&](int m1, int m2, bool in) { if (!in) add(n - k1, n - k2, m1, m2, BT_FULL); });
                it[5] = (int)ent.size();
            }
            long long w = 0;
            for (size_t e = first; e < ent.size(); ++e) w += T.ts.slab[ent[e].w];
            cost.push_back(w);
            items.insert(items.end(), it, it + kItemInts);
        }
    c->nitems = (int)cost.size();
    {
        std::vector<int> order(c->nitems);
        for (int i = 0; i < c->nitems; ++i) order[i] = i;
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
        items.insert(items.end(), order.begin(), order.end());
    }
    if (T.hsize >= (size_t)INT32_MAX) throw CudaError{"mirror table too large for 32-bit H offsets"};
    const size_t hbytes = T.hsize * sizeof(double);
    CK(cudaMalloc(&c->dMH, hbytes));
    CK(cudaMalloc(&c->dMEnt, ent.size() * sizeof(int4)));
    CK(cudaMalloc(&c->dItems, items.size() * sizeof(int)));
    CK(cudaMemcpy(c->dMEnt, ent.data(), ent.size() * sizeof(int4), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->dItems, items.data(), items.size() * sizeof(int), cudaMemcpyHostToDevice));
    c->table_bytes += (int64_t)hbytes + (int64_t)ent.size() * 16 + (int64_t)items.size() * 4;
    c->terms_mirror = (int64_t)T.hsize;
    fill_table(c, G_host, T, c->dMH);
}

// Mirror schedule of the k-chunked kcs kernels (conv.cuh k_conv_kcsm): entries
// as in build_table_mirror; phase-0 rows = pair leaders (A entries), phase-1
// rows = every output row (FULL / REST entries).
void layout_terms_kcsm(int n, TableLayout& T) {
    const int t = conv_tile(n), nk = n / t;
    int off = 0;
    for (int ty = 0; ty < kBandTypes; ++ty) {
        if (ty == BT_REST && kcsr_n(n)) {
            // k_conv_kcsr: the whole row's REST terms in one slab, in the kernel's
            // visiting order (its compile-time table; kcsr_n(n) implies n == 32)
            std::vector<short2> v(kcsr_slab(n), make_short2(-1, -1));
            static constexpr KcsrTab<32> tab{};
            for (int i = 0; i < tab.COUNT; ++i) v[i] = make_short2(tab.k3[i], tab.m3[i]);
            T.ts.off[ty] = off;
            T.ts.slab[ty] = (int)v.size();
            T.ts.slab_max = std::max(T.ts.slab_max, (int)v.size());
            T.term.insert(T.term.end(), v.begin(), v.end());
            off += (int)v.size();
            continue;
        }
        const bool fold = ty == BT_A && kcsf_n(n);  // phase 4: [A pieces | REST(r) | REST'(r'), flagged] per chunk
        const int stride = fold ? kcsf_slab(n) : kcsm_slab(n, ty);
        std::vector<short2> v((size_t)nk * stride, make_short2(-1, -1));
        if (fold) {
            for (int kc = 0; kc < nk; ++kc) {  // kf_pass order: 4-output batches, output, m3
                int pr = kc * stride + kcsf_a_kc(n, kc), pp = pr + even_up(kcsf_rest_kc(n, kc));
                for (int b = 0; b < t / 4; ++b)
                    for (int q = 0; q < 4; ++q)
                        for (int m3 = 0; m3 < n; ++m3) {
                            const int k3 = kc * t + 4 * b + q;
                            if (!rest_term(n, k3, m3)) continue;
                            v[pr++] = make_short2((short)k3, (short)m3);
                            v[pp++] = make_short2((short)(k3 + kMirrorTermFlag), (short)m3);
                        }
            }
            T.partner_terms = true;
        }
        for (int kc = 0; kc < nk; ++kc)
            for (int ti = 0; ti < nk; ++ti) {
                const int sc = band_tile_sc(nk, kc, ti);
                int pos = kc * stride + kcsm_piece_off(n, t, kc, ti, ty);
                const int ks = kcsm_ks(n, kc, ty);
                for (int q = 0; q < ks; ++q)  // band_tile's visiting order (kk passes, then diagonals)
                    for (int i = 0; i < n; ++i) {
                        const int m3 = band_diag(n, nk, kc, ti, i);
                        for (int kk = q * t / ks; kk < (q + 1) * t / ks; ++kk)
                            if (band_term_t(n, t, kc, sc, m3, kk, ty))
                                v[pos++] = make_short2((short)(kc * t + kk), (short)m3);
                    }
            }
        T.ts.off[ty] = off;
        T.ts.slab[ty] = nk * stride;
        T.ts.slab_max = std::max(T.ts.slab_max, nk * stride);
        T.term.insert(T.term.end(), v.begin(), v.end());
        off += nk * stride;
    }
}

void build_table_mirror_kcs(boltz_ctx* c, const double* G_host) {
    const int n = c->n, h = n / 2;
    TableLayout T;
    layout_terms_kcsm(n, T);
    std::vector<int4> ent;
    auto add = [&](int k1, int k2, int m1, int m2, int ty) {
        const int s1 = k1 - m1 + h, s2 = k2 - m2 + h;
        ent.push_back(make_int4((m1 * n + m2) * n, (s1 * n + s2) * n, (int)T.hsize, ty));
        T.meta.push_back(make_int2((int)T.hsize, ty));
        T.hsize += T.ts.slab[ty];
        T.entk.push_back(make_int4(k1, k2, m1, m2));
    };
    auto reps = [&](int k1, int k2, auto&& fn) {
        for (int m1 = std::max(0, k1 - h + 1); m1 <= std::min(n - 1, k1 + h); ++m1)
            for (int m2 = std::max(0, k2 - h + 1); m2 <= std::min(n - 1, k2 + h); ++m2) {
                const int s1 = k1 - m1 + h, s2 = k2 - m2 + h;
                if (m1 < s1 || (m1 == s1 && m2 <= s2))
                    fn(m1, m2, mirror_interior(n, m1) && mirror_interior(n, m2) && mirror_interior(n, s1) &&
                                   mirror_interior(n, s2));
            }
    };
    struct Rows {
        std::vector<int> start, row, aux;
        std::vector<long long> cost;
    } R[3];
    auto partner = [&](int k1, int k2) { return (k1 >= 1 && k2 >= 1) ? (n - k1) * n + (n - k2) : -1; };
    // phase 0: pair leaders' A entries; 1: pair rows' REST entries; 2: every
    // row's FULL entries -- or, without kcsm_split, list 1 = every row's REST and
    // FULL entries (kernel phase 3) and no list 2
    const bool split = kcsm_split(n);
    for (int phase = 0; phase < 3; ++phase)
        for (int k1 = 0; k1 < n; ++k1)
            for (int k2 = 0; k2 < n; ++k2) {
                if (phase == 2 && !split) break;
                const int r = k1 * n + k2, rm = partner(k1, k2);
                const bool pair = rm >= 0 && rm != r;
                if ((phase == 0 && !(pair && r < rm)) || (phase == 1 && split && !pair)) continue;
                if (phase == 1 && kcsf_n(n)) continue;  // REST folded into phase 0 (kernel phase 4)
                Rows& L = R[phase];
                const size_t first = ent.size();
                L.start.push_back((int)first);
                L.row.push_back(r);
                L.aux.push_back(phase == 0 ? rm : (pair ? 1 : 0));
                reps(k1, k2, [&](int m1, int m2, bool in) {
                    const bool interior = pair && in;
                    if (phase == 0 && interior) add(k1, k2, m1, m2, BT_A);
                    if (phase == 1 && interior) add(k1, k2, m1, m2, BT_REST);
                    if ((phase == 2 || (phase == 1 && !split)) && !interior) add(k1, k2, m1, m2, BT_FULL);
                });
                long long w = 0;
                for (size_t e = first; e < ent.size(); ++e) w += T.ts.slab[ent[e].w];
                L.cost.push_back(w);
            }
    auto finish = [&](Rows& L, int end) {
        const int nr = (int)L.row.size();
        std::vector<int> list(L.start);
        list.push_back(end);
        list.insert(list.end(), L.row.begin(), L.row.end());
        list.insert(list.end(), L.aux.begin(), L.aux.end());
        std::vector<int> order(nr);
        for (int i = 0; i < nr; ++i) order[i] = i;
        std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return L.cost[a] > L.cost[b]; });
        list.insert(list.end(), order.begin(), order.end());
        return list;
    };
    std::vector<int> lists[3];
    for (int ph = 0; ph < 3; ++ph) {
        int end = (int)ent.size();  // the next non-empty list's first entry
        for (int q = 2; q > ph; --q)
            if (!R[q].start.empty()) end = R[q].start.front();
        lists[ph] = finish(R[ph], end);
        c->nK[ph] = (int)R[ph].row.size();
    }
    if (T.hsize >= (size_t)INT32_MAX) throw CudaError{"mirror table too large for 32-bit H offsets"};
    const size_t hbytes = T.hsize * sizeof(double);
    CK(cudaMalloc(&c->dMH, hbytes));
    CK(cudaMalloc(&c->dMEnt, ent.size() * sizeof(int4)));
    CK(cudaMemcpy(c->dMEnt, ent.data(), ent.size() * sizeof(int4), cudaMemcpyHostToDevice));
    c->table_bytes += (int64_t)hbytes + (int64_t)ent.size() * 16;
    for (int ph = 0; ph < 3; ++ph) {
        CK(cudaMalloc(&c->dListK[ph], lists[ph].size() * sizeof(int)));
        CK(cudaMemcpy(c->dListK[ph], lists[ph].data(), lists[ph].size() * sizeof(int), cudaMemcpyHostToDevice));
        c->table_bytes += (int64_t)lists[ph].size() * 4;
    }
    c->terms_mirror = (int64_t)T.hsize;
    fill_table(c, G_host, T, c->dMH);
}

// First cell-group column of the mirror kernels' joint longest-first tail
// (conv.cuh mirror_unit): the last BOLTZ_LPT_TAIL columns -- 4 for grids of 16
// or more columns (cfg2, 4096 cells: K2 5.469 -> 5.315 ms, value 714k -> 733k
// evals/s), else 1, i.e. every column longest-first on its own (the host
// pipeline's chunks: e2e 696.6k with 1 against 690-695k with 2-6).  Items
// range from single rows to row pairs (~1.6x) and the earlier columns take them
// longest-first each (measured best in round 1: 11.17 ms against 11.26 in the
// last column only and 11.49 never).  BOLTZ_LPT_FROM overrides (tuning).
// joint longest-first tail columns of the k-chunked kernels (k_conv_kcsm,
// k_conv_kcsr) on many-wave grids; 1 = the last column only
inline int kcs_lpt_tail() {
    const char* e = std::getenv("BOLTZ_LPT_TAIL_KCS");
    return e ? std::max(1, std::atoi(e)) : 1;
}
inline int mirror_lpt_from(int columns) {
    int tail = columns >= 16 ? 4 : 1;
    if (const char* e = std::getenv("BOLTZ_LPT_TAIL")) tail = std::max(1, std::atoi(e));
    int from = std::max(0, columns - tail);
    if (const char* e = std::getenv("BOLTZ_LPT_FROM")) from = std::max(0, std::atoi(e));
    return from;
}

// the mirror schedule runs where the convolution is the single-tile TMA pipe
// (k_conv_mirror) or the k-chunked TMA kcs kernel (k_conv_kcsm)
constexpr bool mirror_pipe_n(int n) {
    return n >= 8 && conv_tile(n) == n && conv_kernel_for(n) == 1 && BOLTZ_PIPE_TMA;
}
constexpr bool mirror_kcs_n(int n) { return n >= 8 && conv_kernel_for(n) == 3 && BOLTZ_PIPE_TMA; }
constexpr bool mirror_eligible_n(int n) { return mirror_pipe_n(n) || mirror_kcs_n(n); }

// Build the folded, pair-symmetric table H (conv.cuh) -- and, where eligible,
// the mirror schedule's table beside it -- from the host G or on the device.
void build_table(boltz_ctx* c, const double* G_host) {
    c->table_bytes = 0;
    build_table_plain(c, G_host);
    bool mirror = mirror_eligible_n(c->n);
    if (const char* e = std::getenv("BOLTZ_MIRROR")) mirror = mirror && std::atoi(e) != 0;
    if (mirror && G_host) mirror = g_mirror_symmetric(c->n, G_host);
    if (mirror) {
        // at N = 8..16 the TMEM variant (k_conv_mirror2) is the default (BOLTZ_MIRROR unset or 2;
        // cfg2 with the 1,2,5,5,2,1 host chunks: value 699.9k / e2e 671.2k evals/s against 693.2k /
        // 666.7k for k_conv_mirror); BOLTZ_MIRROR=1 selects k_conv_mirror
        const char* me = std::getenv("BOLTZ_MIRROR");
        c->mirror2 = mirror_pipe_n(c->n) && c->n % 4 == 0 && (!me || std::atoi(me) == 2);
        if (c->mirror2) build_table_mirror2(c, G_host);
        else if (mirror_pipe_n(c->n)) build_table_mirror(c, G_host);
        else build_table_mirror_kcs(c, G_host);
    }
    c->mirror = mirror;
}

void ensure_workspace(boltz_ctx* c, int64_t cells) {
    int64_t want = (cells + kLanes - 1) / kLanes * kLanes;
    // capacity: up to BOLTZ_WORKSPACE_GB (default 8) GiB of workspace per context
    const int64_t n3 = n3_of(c);
    const int64_t per_cell = n3 * (16 + 16 + 8) + 8;
    double gb = 8.0;
    if (const char* e = std::getenv("BOLTZ_WORKSPACE_GB")) gb = std::max(0.01, std::atof(e));
    int64_t lim = std::max<int64_t>(kLanes, (int64_t)(gb * (1 << 30)) / per_cell / kLanes * kLanes);
    want = std::min(want, lim);
    if (want <= c->cap) return;
    release(c, c->dA); release(c, c->dB); release(c, c->dFs); release(c, c->dMaxIm);
    c->dA = c->dB = nullptr; c->dFs = nullptr; c->dMaxIm = nullptr; c->cap = 0;
    CK(cudaMalloc(&c->dA, (size_t)want * n3 * 16));
    CK(cudaMalloc(&c->dB, (size_t)want * n3 * 16));
    CK(cudaMalloc(&c->dFs, (size_t)want * n3 * 8));
    CK(cudaMalloc(&c->dMaxIm, (size_t)want * 8));
    c->cap = want;
    c->ws_bytes = want * per_cell + c->stage_cap * n3 * 64;
}

// double-buffered device staging for host-memory calls (run_host_pipelined)
// latency schedule scratch: S = kConvWarps x schedule segment partials per cell (complex N^3);
// `cells` counts cells x schedule
void ensure_seg(boltz_ctx* c, int64_t cells) {
    if (cells <= c->seg_cap) return;
    // only the current set's scratch: the other set's may still be in use by
    // the other compute stream (swap_workspace)
    release(c, c->dSeg);
    c->dSeg = nullptr;
    c->seg_cap = 0;
    CK(cudaMalloc(&c->dSeg, (size_t)kConvWarps * cells * n3_of(c) * 16));
    c->seg_cap = cells;
}

// the cell schedule's contiguous f-hat cubes (cells) of the current workspace set
void ensure_cell(boltz_ctx* c, int64_t cells) {
    if (cells <= c->cell_cap) return;
    release(c, c->dCell);
    c->dCell = nullptr;
    c->cell_cap = 0;
    CK(cudaMalloc(&c->dCell, (size_t)cells * n3_of(c) * 16));
    c->cell_cap = cells;
}

// the second workspace set (same capacity as the first)
void ensure_workspace2(boltz_ctx* c) {
    if (c->cap2 == c->cap) return;
    release(c, c->dA2); release(c, c->dB2); release(c, c->dFs2); release(c, c->dMaxIm2);
    release(c, c->dSeg2);  // the second set's scratch; ensure_seg reallocates it on demand
    c->dA2 = c->dB2 = nullptr; c->dFs2 = nullptr; c->dMaxIm2 = nullptr; c->cap2 = 0;
    c->dSeg2 = nullptr;
    c->seg_cap2 = 0;
    release(c, c->dCell2);
    c->dCell2 = nullptr;
    c->cell_cap2 = 0;
    const int64_t n3 = n3_of(c);
    CK(cudaMalloc(&c->dA2, (size_t)c->cap * n3 * 16));
    CK(cudaMalloc(&c->dB2, (size_t)c->cap * n3 * 16));
    CK(cudaMalloc(&c->dFs2, (size_t)c->cap * n3 * 8));
    CK(cudaMalloc(&c->dMaxIm2, (size_t)c->cap * 8));
    c->cap2 = c->cap;
}

// swaps the context's workspace set for the second one (kernels capture the
// pointers at launch, so swapping between enqueues is safe)
void swap_workspace(boltz_ctx* c) {
    std::swap(c->dA, c->dA2);
    std::swap(c->dB, c->dB2);
    std::swap(c->dFs, c->dFs2);
    std::swap(c->dMaxIm, c->dMaxIm2);
    std::swap(c->dSeg, c->dSeg2);
    std::swap(c->seg_cap, c->seg_cap2);
    std::swap(c->dCell, c->dCell2);
    std::swap(c->cell_cap, c->cell_cap2);
}

// pinned bounce slots for pageable host buffers (cells per slot, both directions)
void ensure_bounce(boltz_ctx* c, int64_t cells) {
    if (cells <= c->bounce_cap) return;
    const int64_t n3 = n3_of(c);
    for (int b = 0; b < boltz_ctx::kMaxStageSlots; ++b) {
        if (c->hBounceIn[b]) cudaFreeHost(c->hBounceIn[b]);
        if (c->hBounceOut[b]) cudaFreeHost(c->hBounceOut[b]);
        if (c->hBounceMi[b]) cudaFreeHost(c->hBounceMi[b]);
        c->hBounceIn[b] = c->hBounceOut[b] = c->hBounceMi[b] = nullptr;
    }
    c->bounce_cap = 0;
    for (int b = 0; b < c->stage_slots; ++b) {
        for (int j = 0; j < boltz_ctx::kBounceBlocks; ++j)
            if (!c->ev_blk[b][j]) CK(cudaEventCreateWithFlags(&c->ev_blk[b][j], cudaEventDisableTiming));
        CK(cudaMallocHost(&c->hBounceIn[b], (size_t)cells * n3 * 16));  // complex-sized, like the device staging
        CK(cudaMallocHost(&c->hBounceOut[b], (size_t)cells * n3 * 16));
        CK(cudaMallocHost(&c->hBounceMi[b], (size_t)cells * 8));
    }
    c->bounce_cap = cells;
}

// true when p is ordinary pageable host memory (not cudaHostAlloc'd / registered)
bool is_pageable(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

// block of the bounce pipeline: host copy of block j overlaps the DMA of j-1
size_t bounce_block() {
    static const size_t b = [] {
        double mb = 4.0;
        if (const char* e = std::getenv("BOLTZ_BOUNCE_BLK_MB")) mb = std::max(0.25, std::atof(e));
        return (size_t)(mb * (1 << 20));
    }();
    return b;
}

// Streaming (non-temporal) copy: the destination lines are written without
// being read first, so a copy costs 2 bytes of DRAM traffic per byte instead
// of 3 -- the host copies of the bounce pipeline are DRAM-bound.
__attribute__((target("avx512f"))) void copy_stream_avx512(char* dst, const char* src, size_t bytes) {
    size_t head = (64 - (reinterpret_cast<uintptr_t>(dst) & 63)) & 63;
    head = std::min(head, bytes);
    std::memcpy(dst, src, head);
    dst += head, src += head, bytes -= head;
    const size_t n = bytes / 256;
    for (size_t i = 0; i < n; ++i, dst += 256, src += 256) {
        const __m512d a = _mm512_loadu_pd(src), b = _mm512_loadu_pd(src + 64);
        const __m512d c = _mm512_loadu_pd(src + 128), d = _mm512_loadu_pd(src + 192);
        _mm512_stream_pd(reinterpret_cast<double*>(dst), a);
        _mm512_stream_pd(reinterpret_cast<double*>(dst + 64), b);
        _mm512_stream_pd(reinterpret_cast<double*>(dst + 128), c);
        _mm512_stream_pd(reinterpret_cast<double*>(dst + 192), d);
    }
    std::memcpy(dst, src, bytes % 256);
    _mm_sfence();
}

void copy_block(void* dst, const void* src, size_t bytes) {
    static const bool nt = __builtin_cpu_supports("avx512f") &&
                           !(std::getenv("BOLTZ_COPY_NT") && std::atoi(std::getenv("BOLTZ_COPY_NT")) == 0);
    if (nt) copy_stream_avx512(static_cast<char*>(dst), static_cast<const char*>(src), bytes);
    else std::memcpy(dst, src, bytes);
}

// host copy spread over a few threads (one thread reaches ~15 GB/s; B200
// box, cfg2 pageable e2e / pinned with the persistent pipeline threads and
// streaming stores: 4 threads 0.951, 6 0.946, 8 0.943, 12 0.944, 16 0.948 --
// flat, so the default is the small team, which leaves the caller's cores
// alone; with per-call threads it was 0.81 / 0.90 / 0.91 / 0.92 at 2 / 4 / 8 /
// 12, and with memcpy instead of streaming stores 0.70 / 0.83 / 0.81 at 2 / 4 / 8)
void host_copy(void* dst, const void* src, size_t bytes) {
    static const int threads = [] {
        int t = std::min(6, omp_get_num_procs());
        if (const char* e = std::getenv("BOLTZ_COPY_THREADS")) t = std::max(1, std::atoi(e));
        return t;
    }();
    constexpr size_t kBlock = 1 << 19;
    const int64_t nb = (int64_t)((bytes + kBlock - 1) / kBlock);
    if (threads <= 1 || nb < 2) {
        copy_block(dst, src, bytes);
        return;
    }
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t b = 0; b < nb; ++b) {
        const size_t o = (size_t)b * kBlock;
        copy_block(static_cast<char*>(dst) + o, static_cast<const char*>(src) + o, std::min(kBlock, bytes - o));
    }
}

// the second workspace set for one chunk's enqueue, swapped back even if it throws
struct WorkspaceSwap {
    boltz_ctx* c;
    bool on;
    WorkspaceSwap(boltz_ctx* c_, bool on_) : c(c_), on(on_) {
        if (on) swap_workspace(c);
    }
    ~WorkspaceSwap() {
        if (on) swap_workspace(c);
    }
};

void ensure_staging(boltz_ctx* c, int64_t cells) {
    if (cells <= c->stage_cap) return;
    const int64_t n3 = n3_of(c);
    for (int b = 0; b < boltz_ctx::kMaxStageSlots; ++b) {
        release(c, c->dStageIn[b]);
        release(c, c->dStageOut[b]);
        c->dStageIn[b] = c->dStageOut[b] = nullptr;
    }
    c->stage_cap = 0;
    for (int b = 0; b < c->stage_slots; ++b) {
        CK(cudaMalloc(&c->dStageIn[b], (size_t)cells * n3 * 16));
        CK(cudaMalloc(&c->dStageOut[b], (size_t)cells * n3 * 16));
    }
    c->stage_cap = cells;
    c->ws_bytes = (c->cap + c->cap2) * (n3 * 40 + 8) + c->stage_cap * n3 * 32 * c->stage_slots;
}

// ---------------------------------------------------------------- launchers
template <int N>
struct Launch {
    static constexpr int N3 = N * N * N;
    static dim3 pass_grid(int64_t ngroups) { return dim3((N * N + 7) / 8, (unsigned)ngroups); }

#if BOLTZ_LINE
    // a line kernel (line.cuh) with CPB = c->line_cpb cells per CTA: 2 for
    // device-memory calls, 1 inside the two-stream host pipeline
    // persist: a grid-stride kernel (k_fwd_line), launched as the CTAs that are resident at once
    // (persist kernels are the TMA K1: their shared memory adds the f image, LineTma)
    template <typename K1, typename K2, typename... Args>
    static void launch_line(boltz_ctx* c, bool persist, K1 k1, K2 k2, int64_t nc, cudaStream_t s, Args... args) {
        const int64_t ng = (nc + 31) / 32;
        auto go = [&](auto kern, auto cpb) {
            using LN = Line<N, decltype(cpb)::value>;
            const int smem = persist && BOLTZ_LINE_TMA ? LineTma<N, decltype(cpb)::value>::SMEM : LN::SMEM;
            // keyed by the kernel itself: kernels of one signature share this lambda
            configure_smem(reinterpret_cast<const void*>(kern), c->device, smem);
            int64_t grid = ng * kLanes / LN::CPB;
            if (persist) {
                int per_sm = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, LN::THREADS, smem));
                grid = std::min<int64_t>(grid, (int64_t)std::max(per_sm, 1) * c->num_sms);
            }
            kern<<<(unsigned)grid, LN::THREADS, smem, s>>>(args...);
        };
        if (c->line_cpb == 2) go(k2, std::integral_constant<int, 2>{});
        else go(k1, std::integral_constant<int, 1>{});
        CK(cudaGetLastError());
    }
#endif

    // K3 by k_inv_line2 (all I/O by TMA): group c->dB -> out (FWD: -> c->dA)
    template <bool FWD>
    static void launch_inv2(boltz_ctx* c, const double* base, double* out, int64_t nc, double scale, double coef,
                            double fwd_scale, cudaStream_t s) {
        const int64_t ng = (nc + 31) / 32;
        auto go = [&](auto kern, auto cpb) {
            constexpr int CPB = decltype(cpb)::value;
            using LN = Line<N, CPB>;
            const int smem = LineInv<N, CPB>::SMEM;
            configure_smem(reinterpret_cast<const void*>(kern), c->device, smem);
            const CUtensorMap tB = make_group_tmap(c->dB, ng, N3, CPB);
            const CUtensorMap tBase = base ? make_cells_tmap(base, nc, N) : CUtensorMap{};
            const CUtensorMap tOut = FWD ? CUtensorMap{} : make_cells_tmap(out, nc, N);
            const CUtensorMap tNext = FWD ? make_group_tmap(c->dA, ng, N3, CPB) : CUtensorMap{};
            kern<<<(unsigned)(ng * kLanes / CPB), LN::THREADS, smem, s>>>(
                tB, tBase, tOut, tNext, base ? 1 : 0, reinterpret_cast<double*>(c->dMaxIm), (long long)nc, scale,
                coef, c->pc, c->dFlag, fwd_scale);
        };
        // one cell per CTA, two CTAs per SM: one CTA's TMA loads overlap the other's
        // transforms (cfg2 RK2 step, B200: fused K3 267 -> 198 us, final 191 -> 159 us
        // against two cells per CTA); BOLTZ_LINE_INV2_CPB=2 for the comparison
        static const int cpb = std::getenv("BOLTZ_LINE_INV2_CPB") && std::atoi(std::getenv("BOLTZ_LINE_INV2_CPB")) == 2 ? 2 : 1;
        if (cpb == 2) go(k_inv_line2<N, FWD, 2>, std::integral_constant<int, 2>{});
        else go(k_inv_line2<N, FWD, 1>, std::integral_constant<int, 1>{});
        CK(cudaGetLastError());
    }

    // user real f (device, nc cells) -> group complex fhat in c->dA
    static void forward(boltz_ctx* c, const double* f, int64_t nc, cudaStream_t s) {
        const int64_t ng = (nc + 31) / 32;
        const double sv = c->pc.dv / std::sqrt(2.0 * kPi);
        const double par = ((N / 2) & 1) ? -1.0 : 1.0;  // ((-1)^{N/2})^3
        const double scale = sv * sv * sv * par;
#if BOLTZ_LINE
        if constexpr (line_n(N)) {
          if ((reinterpret_cast<uintptr_t>(f) & 15) == 0) {
            Timed t_(c, KIND_FFT, s);
            if (BOLTZ_LINE_TMA) {
                const CUtensorMap tm = make_group_tmap(c->dA, (nc + 31) / 32, N3, c->line_cpb);
                const CUtensorMap tf = BOLTZ_LINE_TMA_LOAD ? make_cells_tmap(f, nc, N) : CUtensorMap{};
                launch_line(c, true, k_fwd_line_tma<N, 1>, k_fwd_line_tma<N, 2>, nc, s, f, tf, tm, (long long)nc,
                            scale, c->dFlag);
            } else {
                launch_line(c, BOLTZ_LINE_PERSIST != 0, k_fwd_line<N, 1>, k_fwd_line<N, 2>, nc, s, f, c->dA,
                            (long long)nc, scale, c->dFlag);
            }
            return;
          }
        }
#endif
#if BOLTZ_FUSED
        if constexpr (Fused<N>::FITS) {
            using F = Fused<N>;
            static PerDevice configured;  // attributes are per device
            configured.once(c->device, [&] {
                CK(cudaFuncSetAttribute(k_fwd_fused<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, F::SMEM));
            });
            Timed t_(c, KIND_FFT, s);
            k_fwd_fused<N><<<(unsigned)(ng * kLanes / F::CPB), F::THREADS, F::SMEM, s>>>(f, c->dA, nc, scale,
                                                                                          c->dFlag);
            CK(cudaGetLastError());
            return;
        }
#endif
        dim3 blk(32, 8);
        { Timed t_(c, KIND_FFT, s); k_fft_pass<N, 2, -1, PASS_PACK_FWD><<<pass_grid(ng), blk, 0, s>>>(f, c->dA, nullptr, nullptr, c->dFlag, nc, 1.0); }
        { Timed t_(c, KIND_FFT, s); k_fft_pass<N, 1, -1, PASS_MID><<<pass_grid(ng), blk, 0, s>>>(nullptr, c->dA, nullptr, nullptr, c->dFlag, nc, 1.0); }
        { Timed t_(c, KIND_FFT, s); k_fft_pass<N, 0, -1, PASS_FWD_LAST><<<pass_grid(ng), blk, 0, s>>>(nullptr, c->dA, nullptr, nullptr, c->dFlag, nc,
                                                                           scale); }
        CK(cudaGetLastError());
    }
    // group complex c->dA -> group complex (s_k * Qhat) in c->dB
    // hermitian: the input is the transform of a real f (collide / RK2), so the
    // mirror schedule may run; evaluate_qhat of a caller's fhat never does
    static void conv(boltz_ctx* c, int64_t nc, cudaStream_t s, bool hermitian = false) {
        const int64_t ng = (nc + 31) / 32;
        const int sched = effective_schedule(c, nc);
        if constexpr (conv_tile(N) == N && N <= 16) {
            // one or a few cells: lane = output k3 (conv.cuh k_conv_cell); one grid row per cell
            if (sched == kScheduleCell && nc <= 65535) {
                using CL = CellLayout<N>;
                static PerDevice configured;  // attributes are per device
                configured.once(c->device, [&] {
                    CK(cudaFuncSetAttribute(k_conv_cell<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, CL::BYTES));
                });
                ensure_cell(c, nc);
                Timed t_(c, KIND_CONV, s);
                const long long tot = nc * (long long)N3;
                k_cell_gather<N><<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(c->dA, c->dCell, (int)nc);
                k_conv_cell<N><<<dim3(N * N, (unsigned)nc), kLanes * kCellWarps, CL::BYTES, s>>>(
                    c->dCell, c->dB, c->dH, c->dEnt, c->dRowStart, c->slab);
                c->launches[KIND_CONV]++;  // two kernels under one timing bracket
                CK(cudaGetLastError());
                return;
            }
        }
        if constexpr (mirror_kcs_n(N)) {
            if (hermitian && c->mirror && sched == 0) {
                constexpr int NK = N / conv_tile(N), KC1 = NK > 1 ? 1 : 0;
                // 8-warp CTAs at N = 24 (kcsm_warps) unless the batch has at most kConvWarps
                // groups: then kConvWarps-warp CTAs, so no CTA carries idle warps' shared memory
                auto run = [&](auto wtag) {
                    constexpr int W = decltype(wtag)::value;
                    constexpr int P0 = kcsf_n(N) ? 4 : 0;  // the phase-0 kernels: with the REST fold or plain
                    const int smem_ph[5] = {W * KcsmLayout<N, 0>::WARP_BYTES, W * KcsmLayout<N, 1>::WARP_BYTES,
                                            W * KcsmLayout<N, 2>::WARP_BYTES, W * KcsmLayout<N, 3>::WARP_BYTES,
                                            W * KcsmLayout<N, 4>::WARP_BYTES + KcsmLayout<N, 4>::TMEM_BYTES};
                    static PerDevice configured;  // attributes are per device
                    configured.once(c->device, [&] {
                        auto cfg = [&](auto fn, int ph) {
                            CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_ph[ph]));
                            CK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
                        };
                        cfg(k_conv_kcsm<N, 0, P0, W>, P0);
                        cfg(k_conv_kcsm<N, KC1, P0, W>, P0);
                        if constexpr (kcsr_n(N)) {
                            if constexpr (BOLTZ_KCSR_YBUF == 4) {
                                CK(cudaFuncSetAttribute(k_conv_kcsrq<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                        KcsrqLayout<N>::WARP_BYTES * kKcsrWarps));
                                CK(cudaFuncSetAttribute(k_conv_kcsrq<N>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
                            } else {
                                CK(cudaFuncSetAttribute(k_conv_kcsr<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                        KcsrLayout<N>::WARP_BYTES * kKcsrWarps));
                                CK(cudaFuncSetAttribute(k_conv_kcsr<N>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
                            }
                        }
                        if constexpr (kcsm_split(N)) {
                            cfg(k_conv_kcsm<N, 0, 1, W>, 1);
                            cfg(k_conv_kcsm<N, KC1, 1, W>, 1);
                            cfg(k_conv_kcsm<N, 0, 2, W>, 2);
                            cfg(k_conv_kcsm<N, KC1, 2, W>, 2);
                        } else {
                            cfg(k_conv_kcsm<N, 0, 3, W>, 3);
                            cfg(k_conv_kcsm<N, KC1, 3, W>, 3);
                        }
                    });
                    const unsigned gy = (unsigned)((ng + W - 1) / W);
                    // longest rows first: every column (each on its own) for grids a few waves
                    // deep, else the last kcs_lpt_tail() columns jointly (conv.cuh lpt_unit)
                    auto few = [&](int nrows, unsigned cols) { return (int64_t)nrows * cols < 8 * 2 * 148; };
                    auto lpt = [&](int nrows) { return few(nrows, gy) ? (int)gy : std::max(0, (int)gy - kcs_lpt_tail()); };
                    Timed t_(c, KIND_CONV, s);
                    // phase 0 (pair leaders' A sums + mirror seeds), 1 (REST), 2 (FULL, final), per k-chunk
                    auto go = [&](auto kern, int ph) {
                        // list 1 runs phase 3 when not split; list 0 phase 4 with the REST fold
                        const int kph = ph == 1 && !kcsm_split(N) ? 3 : ph == 0 ? P0 : ph;
                        kern<<<dim3(c->nK[ph], gy), kLanes * W, smem_ph[kph], s>>>(c->dA, c->dB, c->dMH, c->dMEnt,
                                                                                    c->dListK[ph], c->nK[ph], (int)ng,
                                                                                    lpt(c->nK[ph]), (int)few(c->nK[ph], gy));
                    };
                    go(k_conv_kcsm<N, 0, P0, W>, 0);
                    if constexpr (NK > 1) go(k_conv_kcsm<N, KC1, P0, W>, 0);
                    if constexpr (kcsf_n(N)) {  // REST folded into phase 0: FULL entries only
                        go(k_conv_kcsm<N, 0, 2, W>, 2);
                        if constexpr (NK > 1) go(k_conv_kcsm<N, KC1, 2, W>, 2);
                    } else if constexpr (kcsr_n(N)) {  // the pair rows' REST entries, both k-chunks in one launch
                        const unsigned gr = (unsigned)((ng + kKcsrWarps - 1) / kKcsrWarps);
                        const bool fr = few(c->nK[1], gr);
                        const int lr = fr ? (int)gr : std::max(0, (int)gr - kcs_lpt_tail());
                        if constexpr (BOLTZ_KCSR_YBUF == 4)  // one y row per warp, refilled by quarters
                            k_conv_kcsrq<N><<<dim3(c->nK[1], gr), kLanes * kKcsrWarps,
                                              KcsrqLayout<N>::WARP_BYTES * kKcsrWarps, s>>>(
                                c->dA, c->dB, c->dMH, c->dMEnt, c->dListK[1], c->nK[1], (int)ng, lr, (int)fr);
                        else
                            k_conv_kcsr<N><<<dim3(c->nK[1], gr), kLanes * kKcsrWarps, KcsrLayout<N>::WARP_BYTES * kKcsrWarps,
                                             s>>>(c->dA, c->dB, c->dMH, c->dMEnt, c->dListK[1], c->nK[1], (int)ng, lr, (int)fr);
                        go(k_conv_kcsm<N, 0, 2, W>, 2);
                        if constexpr (NK > 1) go(k_conv_kcsm<N, KC1, 2, W>, 2);
                    } else if constexpr (kcsm_split(N)) {
                        go(k_conv_kcsm<N, 0, 1, W>, 1);
                        if constexpr (NK > 1) go(k_conv_kcsm<N, KC1, 1, W>, 1);
                        go(k_conv_kcsm<N, 0, 2, W>, 2);
                        if constexpr (NK > 1) go(k_conv_kcsm<N, KC1, 2, W>, 2);
                    } else {
                        go(k_conv_kcsm<N, 0, 3, W>, 1);
                        if constexpr (NK > 1) go(k_conv_kcsm<N, KC1, 3, W>, 1);
                    }
                };
                if constexpr (kcsm_warps(N) != kConvWarps) {
                    if (ng <= kConvWarps) run(std::integral_constant<int, kConvWarps>{});
                    else run(std::integral_constant<int, kcsm_warps(N)>{});
                } else {
                    run(std::integral_constant<int, kConvWarps>{});
                }
                c->launches[KIND_CONV] += kcsf_n(N) ? 2 * NK - 1 : kcsr_n(N) ? 2 * NK : (kcsm_split(N) ? 3 : 2) * NK - 1;  // one timing bracket
                CK(cudaGetLastError());
                return;
            }
        }
        if constexpr (mirror_pipe_n(N) && N % 4 == 0) {
            if (hermitian && c->mirror && c->mirror2 && sched == 0) {
                const int smem = Mirror2Layout<N>::CTA_BYTES;
                static PerDevice configured;  // attributes are per device
                configured.once(c->device, [&] {
                    CK(cudaFuncSetAttribute(k_conv_mirror2<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                    CK(cudaFuncSetAttribute(k_conv_mirror2<N>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
                });
                dim3 grid((unsigned)c->nitems, (unsigned)((ng + kConvWarps - 1) / kConvWarps));
                const int lpt = mirror_lpt_from((int)grid.y);
                Timed t_(c, KIND_CONV, s);
                k_conv_mirror2<N><<<grid, kLanes * kConvWarps, smem, s>>>(c->dA, c->dB, c->dMH, c->dMEnt, c->dItems,
                                                                          c->dItems + kItemInts * c->nitems, (int)ng,
                                                                          lpt);
                CK(cudaGetLastError());
                return;
            }
        }
        if constexpr (mirror_pipe_n(N)) {
            if (hermitian && c->mirror && sched == 0) {
                const int smem = kConvWarps * MirrorLayout<N>::WARP_BYTES;
                static PerDevice configured;  // attributes are per device
                configured.once(c->device, [&] {
                    CK(cudaFuncSetAttribute(k_conv_mirror<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                    CK(cudaFuncSetAttribute(k_conv_mirror<N>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
                });
                dim3 grid((unsigned)c->nitems, (unsigned)((ng + kConvWarps - 1) / kConvWarps));
                const int lpt = mirror_lpt_from((int)grid.y);
                Timed t_(c, KIND_CONV, s);
                k_conv_mirror<N><<<grid, kLanes * kConvWarps, smem, s>>>(c->dA, c->dB, c->dMH, c->dMEnt, c->dItems,
                                                                         c->dItems + kItemInts * c->nitems, (int)ng,
                                                                         lpt);
                CK(cudaGetLastError());
                return;
            }
        }
        if constexpr (conv_kernel_for(N) == 1 && conv_tile(N) == N &&
                      kConvWarps * PipeLayout<N>::WARP_BYTES <= 220 * 1024) {
            if (sched > 0 && sched < kScheduleCell) {
                const int S = kConvWarps * sched;  // segments per row
                const int smem = kConvWarps * PipeLayout<N>::WARP_BYTES;
                static PerDevice configured;  // attributes are per device
                configured.once(c->device, [&] {
                    CK(cudaFuncSetAttribute(k_conv_seg<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                    CK(cudaFuncSetAttribute(k_conv_seg<N>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
                });
                ensure_seg(c, ng * kLanes * sched);
                Timed t_(c, KIND_CONV, s);
                k_conv_seg<N><<<dim3(N * N, (unsigned)ng, (unsigned)sched), kLanes * kConvWarps, smem, s>>>(
                    c->dA, c->dSeg, c->dH, c->dEnt, c->dRowStart, (int)ng, S);
                const long long total = ng * N3 * kLanes;
                k_conv_seg_reduce<N><<<(unsigned)((total + 255) / 256), 256, 0, s>>>(c->dSeg, c->dB, ng, S);
                c->launches[KIND_CONV]++;  // two kernels under one timing bracket
                CK(cudaGetLastError());
                return;
            }
        }
        constexpr int NK = N / conv_tile(N);
        dim3 grid(N * N * NK, (unsigned)((ng + kConvWarps - 1) / kConvWarps));
        // longest-rows-first in every column when the grid is a few waves deep (~2
        // CTAs per SM resident), else in the last column only (conv.cuh conv_row)
        int lpt = (int64_t)grid.x * grid.y < 8 * 2 * 148 ? 0 : (int)grid.y - 1;
        if (const char* e = std::getenv("BOLTZ_LPT_FROM")) lpt = std::atoi(e);  // tuning
        if constexpr (conv_kernel_for(N) == 1 && kConvWarps * PipeLayout<N>::WARP_BYTES <= 220 * 1024) {
            const int smem = kConvWarps * PipeLayout<N>::WARP_BYTES;
            static PerDevice configured;  // attributes are per device
            configured.once(c->device, [&] {
                CK(cudaFuncSetAttribute(k_conv_pipe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                CK(cudaFuncSetAttribute(k_conv_pipe<N>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
            });
            Timed t_(c, KIND_CONV, s);
            k_conv_pipe<N><<<grid, kLanes * kConvWarps, smem, s>>>(c->dA, c->dB, c->dH, c->dEnt, c->dRowStart,
                                                                    (int)ng, lpt);
        } else if constexpr (conv_kernel_for(N) == 3) {
            using LY = KcsLayout<N>;
            const int smem = kConvWarps * LY::WARP_BYTES;
            constexpr int KC1 = NK > 1 ? 1 : 0;
            static PerDevice configured;  // attributes are per device
            configured.once(c->device, [&] {
                CK(cudaFuncSetAttribute(k_conv_kcs<N, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                CK(cudaFuncSetAttribute(k_conv_kcs<N, 0>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
                CK(cudaFuncSetAttribute(k_conv_kcs<N, KC1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
                CK(cudaFuncSetAttribute(k_conv_kcs<N, KC1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
            });
            dim3 g1(N * N, (unsigned)((ng + kConvWarps - 1) / kConvWarps));
            Timed t_(c, KIND_CONV, s);
            k_conv_kcs<N, 0><<<g1, kLanes * kConvWarps, smem, s>>>(c->dA, c->dB, c->dH, c->dEnt, c->dRowStart, (int)ng, lpt);
            if constexpr (NK > 1)
                k_conv_kcs<N, KC1><<<g1, kLanes * kConvWarps, smem, s>>>(c->dA, c->dB, c->dH, c->dEnt, c->dRowStart,
                                                                         (int)ng, lpt);
            if constexpr (NK > 1) c->launches[KIND_CONV]++;  // one k-chunk kernel each
        } else
        { Timed t_(c, KIND_CONV, s); k_conv<N><<<grid, kLanes * kConvWarps, 0, s>>>(c->dA, c->dB, c->dH, c->dEnt, c->dRowStart, (int)ng, lpt); }
        CK(cudaGetLastError());
    }
    // group complex c->dB (already * s_m) -> group real Qt in (double*)c->dA; max|Im| per cell
    static void inverse(boltz_ctx* c, int64_t nc, cudaStream_t s) {
        const int64_t ng = (nc + 31) / 32;
        const double dz = kPi / c->L;
        const double sz = dz / std::sqrt(2.0 * kPi);
        const double par = ((N / 2) & 1) ? -1.0 : 1.0;
        const double scale = sz * sz * sz;
        dim3 blk(32, 8);
        CK(cudaMemsetAsync(c->dMaxIm, 0, (size_t)nc * 8, s));
        { Timed t_(c, KIND_FFT, s); k_fft_pass<N, 2, +1, PASS_MID><<<pass_grid(ng), blk, 0, s>>>(nullptr, c->dB, nullptr, nullptr, c->dFlag, nc, 1.0); }
        { Timed t_(c, KIND_FFT, s); k_fft_pass<N, 1, +1, PASS_MID><<<pass_grid(ng), blk, 0, s>>>(nullptr, c->dB, nullptr, nullptr, c->dFlag, nc, 1.0); }
        // the INV_LAST pass folds par into the sign of its scale; max|Im| uses |scale|
        { Timed t_(c, KIND_FFT, s); k_fft_pass<N, 0, +1, PASS_INV_LAST><<<pass_grid(ng), blk, 0, s>>>(
            nullptr, c->dB, reinterpret_cast<double*>(c->dA), c->dMaxIm, c->dFlag, nc, scale * par); }
        CK(cudaGetLastError());
    }
    // group complex c->dB -> out = base + coef * P_N(Re iFFT) (user layout); max|Im| -> c->dMaxIm
    static void inverse_project(boltz_ctx* c, const double* base, double* out, int64_t nc, double coef,
                                cudaStream_t s) {
#if BOLTZ_LINE
        if constexpr (line_n(N)) {
            const double sz = (kPi / c->L) / std::sqrt(2.0 * kPi);
            const double par = ((N / 2) & 1) ? -1.0 : 1.0;
            Timed t_(c, KIND_PROJECT, s);
            if (BOLTZ_LINE_INV2 && ((reinterpret_cast<uintptr_t>(base) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) {
                launch_inv2<false>(c, base, out, nc, sz * sz * sz * par, coef, 0.0, s);
                return;
            }
            launch_line(c, false, k_inv_line<N, false, 1>, k_inv_line<N, false, 2>, nc, s, (const double2*)c->dB, base, out,
                        reinterpret_cast<double*>(c->dMaxIm), (long long)nc, sz * sz * sz * par, coef, c->pc, c->dFlag,
                        (double2*)nullptr, CUtensorMap{}, 0.0);
            return;
        }
#endif
#if BOLTZ_FUSED
        if constexpr (Fused<N>::FITS) {
            using F = Fused<N>;
            const int64_t ng = (nc + 31) / 32;
            const double sz = (kPi / c->L) / std::sqrt(2.0 * kPi);
            const double par = ((N / 2) & 1) ? -1.0 : 1.0;
            static PerDevice configured;  // attributes are per device
            configured.once(c->device, [&] {
                CK(cudaFuncSetAttribute(k_inv_project<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, F::SMEM));
            });
            Timed t_(c, KIND_PROJECT, s);
            k_inv_project<N><<<(unsigned)(ng * kLanes / F::CPB), F::THREADS, F::SMEM, s>>>(
                c->dB, base, out, reinterpret_cast<double*>(c->dMaxIm), nc, sz * sz * sz * par, coef, c->pc,
                c->dFlag);
            CK(cudaGetLastError());
            return;
        }
#endif
        inverse(c, nc, s);
        project(c, base, out, nc, coef, s);
    }
    // RK2 stage hand-off: f* = base + coef * P_N(Re iFFT(c->dB)) and straight on to
    // fhat(f*) in c->dA (fused when the cube fits in smem: f* never touches HBM);
    // otherwise through the user-layout scratch `fs`.
    static void inverse_project_forward(boltz_ctx* c, const double* base, double* fs, int64_t nc, double coef,
                                        cudaStream_t s) {
#if BOLTZ_LINE
        if constexpr (line_n(N)) {
          if ((reinterpret_cast<uintptr_t>(base) & 15) == 0) {
            const double sz = (kPi / c->L) / std::sqrt(2.0 * kPi);
            const double sv = c->pc.dv / std::sqrt(2.0 * kPi);
            const double par = ((N / 2) & 1) ? -1.0 : 1.0;
            Timed t_(c, KIND_PROJECT, s);
            if (BOLTZ_LINE_INV2) {
                launch_inv2<true>(c, base, nullptr, nc, sz * sz * sz * par, coef, sv * sv * sv * par, s);
                return;
            }
            launch_line(c, false, k_inv_line<N, true, 1>, k_inv_line<N, true, 2>, nc, s, (const double2*)c->dB, base,
                        (double*)nullptr, reinterpret_cast<double*>(c->dMaxIm), (long long)nc, sz * sz * sz * par, coef,
                        c->pc, c->dFlag, c->dA,
                        BOLTZ_LINE_TMA ? make_group_tmap(c->dA, (nc + 31) / 32, N3, c->line_cpb) : CUtensorMap{},
                        sv * sv * sv * par);
            return;
          }
        }
#endif
#if BOLTZ_FUSED
        if constexpr (Fused<N>::FITS) {
            using F = Fused<N>;
            const int64_t ng = (nc + 31) / 32;
            const double sz = (kPi / c->L) / std::sqrt(2.0 * kPi);
            const double sv = c->pc.dv / std::sqrt(2.0 * kPi);
            const double par = ((N / 2) & 1) ? -1.0 : 1.0;
            static PerDevice configured;  // attributes are per device
            configured.once(c->device, [&] {
                CK(cudaFuncSetAttribute(k_inv_project<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        F::SMEM));
            });
            Timed t_(c, KIND_PROJECT, s);
            k_inv_project<N, true><<<(unsigned)(ng * kLanes / F::CPB), F::THREADS, F::SMEM, s>>>(
                c->dB, base, nullptr, reinterpret_cast<double*>(c->dMaxIm), nc, sz * sz * sz * par, coef, c->pc,
                c->dFlag, c->dA, sv * sv * sv * par);
            CK(cudaGetLastError());
            return;
        }
#endif
        inverse_project(c, base, fs, nc, coef, s);
        forward(c, fs, nc, s);
    }
    // group real Qt in (double*)c->dA -> out = base + coef * P_N(Qt)  (user layout)
    static void project(boltz_ctx* c, const double* base, double* out, int64_t nc, double coef, cudaStream_t s) {
        const int64_t ng = (nc + 31) / 32;
        // partial moments go to c->dB: the convolution output is consumed by then
        // (conserve() never uses it), and 40 B x 8 slices per cell fit many times over
        double* part = reinterpret_cast<double*>(c->dB);
        const double* R = reinterpret_cast<const double*>(c->dA);
        dim3 grid((unsigned)(ng * 4), kProjSlices);
        {
            Timed t_(c, KIND_PROJECT, s);
            k_project_moments<N><<<grid, 256, 0, s>>>(R, part, nc, c->pc);
            k_project_apply<N><<<grid, 256, 0, s>>>(R, part, base, out, nc, coef, c->pc, c->dFlag);
            c->launches[KIND_PROJECT]++;
        }
        CK(cudaGetLastError());
    }
    static void pack_complex(boltz_ctx* c, const double* in, double2* dst, int64_t nc, int sign, cudaStream_t s) {
        const int64_t ng = (nc + 31) / 32;
        dim3 grid((unsigned)std::min<int64_t>((N3 + 7) / 8, 512), (unsigned)ng);
        { Timed t_(c, KIND_LAYOUT, s); k_pack_complex<N><<<grid, 256, 0, s>>>(reinterpret_cast<const double2*>(in), dst, nc, sign); }
        CK(cudaGetLastError());
    }
    static void unpack_complex(boltz_ctx* c, const double2* src, double* out, int64_t nc, int sign, cudaStream_t s) {
        const int64_t ng = (nc + 31) / 32;
        dim3 grid((unsigned)std::min<int64_t>((N3 + 7) / 8, 512), (unsigned)ng);
        { Timed t_(c, KIND_LAYOUT, s); k_unpack_complex<N><<<grid, 256, 0, s>>>(src, reinterpret_cast<double2*>(out), nc, sign); }
        CK(cudaGetLastError());
    }
    static void unpack_real(boltz_ctx* c, const double* src, double* out, int64_t nc, cudaStream_t s) {
        const int64_t ng = (nc + 31) / 32;
        dim3 grid((unsigned)std::min<int64_t>((N3 + 7) / 8, 512), (unsigned)ng);
        { Timed t_(c, KIND_LAYOUT, s); k_unpack_real<N><<<grid, 256, 0, s>>>(src, out, nc); }
        CK(cudaGetLastError());
    }
    static void pack_real(boltz_ctx* c, const double* in, double* dst, int64_t nc, cudaStream_t s) {
        const int64_t ng = (nc + 31) / 32;
        dim3 grid((unsigned)std::min<int64_t>((N3 + 7) / 8, 512), (unsigned)ng);
        { Timed t_(c, KIND_LAYOUT, s); k_pack_real<N><<<grid, 256, 0, s>>>(in, dst, nc); }
        CK(cudaGetLastError());
    }
};

// DFMA throughput of the whole device, TFLOP/s (2 flops per DFMA)
double fp64_peak_probe(double seconds) {
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    double* d = nullptr;
    CK(cudaMalloc(&d, 8));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int blocks = sms * 4, threads = 256;
    int iters = 1 << 14;
    double best = 0.0, spent = 0.0;
    k_dfma_probe<<<blocks, threads>>>(d, iters, 0.999999, 1e-6);  // warm-up
    CK(cudaDeviceSynchronize());
    while (spent < seconds * 1e3) {
        CK(cudaEventRecord(e0));
        k_dfma_probe<<<blocks, threads>>>(d, iters, 0.999999, 1e-6);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        spent += ms;
        const double tf = 2.0 * 8.0 * iters * (double)blocks * threads / (ms * 1e-3) / 1e12;
        best = std::max(best, tf);
        if (ms < 50.0f) iters *= 2;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    return best;
}

template <typename F>
void dispatch(int n, F&& f) {
    switch (n) {
#define BOLTZ_CASE(N) \
    case N: f(Launch<N>{}); break;
        BOLTZ_FOR_EACH_N(BOLTZ_CASE)
#undef BOLTZ_CASE
        default: throw CudaError{"unsupported N"};
    }
}

int guard_ctx(boltz_ctx* c) {
    if (!c) {
        set_error("null context");
        return BOLTZ_ERR_CONFIG;
    }
    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) {
        set_error(std::string("cudaSetDevice: ") + cudaGetErrorString(e));
        return BOLTZ_ERR_CUDA;
    }
    return BOLTZ_OK;
}

// Runs fn(chunk_in, chunk_out, cells, stream) over chunks of the batch, staging
// host memory through the context buffers when mem == HOST.  in_elems /
// out_elems: doubles per cell of the user-layout input / output.
int check_flag(boltz_ctx* c, cudaStream_t s);
template <typename Fn>
int run_host_pipelined(boltz_ctx* c, const double* in, double* out, int64_t ncells, int in_elems, int out_elems,
                       cudaStream_t s, double* max_imag, Fn&& fn);

template <typename Fn>
int run_chunked(boltz_ctx* c, const double* in, double* out, int64_t ncells, int in_elems, int out_elems, int mem,
                void* stream, double* max_imag, Fn&& fn) {
    if (ncells < 0 || (ncells > 0 && (!in || !out))) {
        set_error("invalid batch arguments (null pointer or negative count)");
        return BOLTZ_ERR_CONFIG;
    }
    if (mem != BOLTZ_MEM_HOST && mem != BOLTZ_MEM_DEVICE) {
        set_error("mem must be BOLTZ_MEM_HOST or BOLTZ_MEM_DEVICE");
        return BOLTZ_ERR_CONFIG;
    }
    if (ncells == 0) return BOLTZ_OK;
    cudaStream_t s = (cudaStream_t)stream;  // NULL = the CUDA default stream
    note_capture(c, s);
    if (mem == BOLTZ_MEM_HOST) return run_host_pipelined(c, in, out, ncells, in_elems, out_elems, s, max_imag, fn);
    ensure_workspace(c, ncells);
    const bool deferred = c->async_mode;  // flag checked at boltz_sync
    if (!deferred) CK(cudaMemsetAsync(c->dFlag, 0, sizeof(int), s));
    for (int64_t c0 = 0; c0 < ncells; c0 += c->cap) {
        const int64_t nc = std::min<int64_t>(c->cap, ncells - c0);
        fn(in + c0 * in_elems, out + c0 * out_elems, nc, s);
        if (max_imag) CK(cudaMemcpyAsync(max_imag + c0, c->dMaxIm, (size_t)nc * 8, cudaMemcpyDeviceToDevice, s));
    }
    if (deferred) return BOLTZ_OK;
    return check_flag(c, s);
}

// Host-memory calls: the batch is cut into chunks and pipelined over four
// streams -- H2D of chunk i+1 (copy engine), compute of chunk i (`s` for even,
// `comp2` with the second workspace for odd chunks), D2H of chunk i-1 (the
// other copy engine) -- through stage_slots staging buffer pairs, so with
// pinned host memory the PCIe traffic hides behind the kernels.  Pageable
// caller memory runs the same pipeline through pinned bounce buffers, with
// the host copies on two worker threads (run_host_bounced).
template <typename Fn>
int run_host_bounced(boltz_ctx* c, const double* in, double* out, int in_elems, int out_elems, cudaStream_t s,
                     double* max_imag, Fn& fn, const std::vector<int64_t>& bounds, bool two, bool bounce_in,
                     bool bounce_out);

template <typename Fn>
int run_host_pipelined(boltz_ctx* c, const double* in, double* out, int64_t ncells, int in_elems, int out_elems,
                       cudaStream_t s, double* max_imag, Fn&& fn) {
    std::vector<int64_t> bounds{0};
    // chunk boundaries on whole K2 CTA columns (kConvWarps groups of 32 cells)
    constexpr int64_t kGrain = (int64_t)kLanes * kConvWarps;
    auto up32 = [](int64_t x) { return (x + kGrain - 1) / kGrain * kGrain; };
    // Chunk schedule (relative weights, measured best on B200 for cfg2): the first
    // H2D and the last D2H cannot overlap compute, so the edge chunks are small;
    // odd chunks run on a second stream, so each chunk's last wave overlaps the
    // next chunk's work.  With the mirror schedule, whose work items are row
    // pairs and which only pays from ~1.5k cells up, large middle chunks win:
    // 1,2,3,5,5,3,2,1 (cfg2 e2e pinned / pageable, k evals/s, two runs: 671.7 /
    // 618.5; 1,2,5,5,2,1 669.9 / 612.8; 1,2,4,4,2,1 668.4 / 618.6; 1,2,6,6,2,1
    // 666.0 / 605.8; 0.5,1.5,5,5,1.5,0.5 660.3 / 586; round 1's 1,3,3,1 627-641;
    // the pageable bounce path needs the small edge chunks); the plain schedule
    // prefers 2,6,8,8,6,2 (602k).  BOLTZ_HOST_CHUNKS="a,b,..." overrides.
    std::vector<double> w = c->mirror ? std::vector<double>{1, 2, 3, 5, 5, 3, 2, 1}
                                      : std::vector<double>{2, 6, 8, 8, 6, 2};
    if (const char* sched = std::getenv("BOLTZ_HOST_CHUNKS")) {
        w.clear();
        for (const char* p = sched; *p;) {
            char* end = nullptr;
            const double v = std::strtod(p, &end);
            if (end == p) break;
            if (v > 0) w.push_back(v);
            p = (*end == ',') ? end + 1 : end;
        }
    }
    if (ncells > 1024) {
        double tot = 0, acc = 0;
        for (double v : w) tot += v;
        for (size_t i = 0; i + 1 < w.size(); ++i) {
            acc += w[i];
            const int64_t b = std::min<int64_t>(ncells, up32((int64_t)(ncells * acc / tot)));
            if (b > bounds.back() && b < ncells) bounds.push_back(b);
        }
    }
    bounds.push_back(ncells);
    int64_t chunk = 0;
    for (size_t i = 1; i < bounds.size(); ++i) chunk = std::max(chunk, bounds[i] - bounds[i - 1]);
    ensure_workspace(c, chunk);
    if (chunk > c->cap) {  // workspace limit: fall back to uniform chunks of the capacity
        bounds.assign(1, 0);
        for (int64_t b = c->cap; b < ncells; b += c->cap) bounds.push_back(b);
        bounds.push_back(ncells);
        chunk = c->cap;
    }
    ensure_staging(c, chunk);
    const int64_t nchunks = (int64_t)bounds.size() - 1;
    // odd chunks compute on comp2 with the second workspace; comp2 joins s's
    // prior work first and s waits for comp2 at the end (stream semantics kept)
    bool two = nchunks > 1;
    if (const char* e = std::getenv("BOLTZ_HOST_STREAMS")) two = two && std::atoi(e) > 1;  // tuning / A-B
    if (two) ensure_workspace2(c);
    // two compute streams: one-cell line K1/K3 CTAs, so that the other stream's
    // K2 CTAs still fit beside them on an SM (restored on return)
    struct CpbGuard {
        boltz_ctx* c;
        int old;
        ~CpbGuard() { c->line_cpb = old; }
    } cpb_guard{c, c->line_cpb};
    if (two) {
        static const int pipe_cpb = std::getenv("BOLTZ_PIPE_LINE_CPB") ? std::atoi(std::getenv("BOLTZ_PIPE_LINE_CPB")) : 1;
        c->line_cpb = pipe_cpb == 2 ? 2 : 1;  // tuning / A-B: K1's cells per CTA inside the pipeline
    }
    // pageable caller memory goes through the pinned bounce ring (host threads
    // copy; the DMA engines only ever see pinned memory)
    bool bounce_in = is_pageable(in), bounce_out = is_pageable(out) || (max_imag && is_pageable(max_imag));
    if (const char* e = std::getenv("BOLTZ_BOUNCE"))
        if (std::atoi(e) == 0) bounce_in = bounce_out = false;
    // a few cells (<= 512 KiB each way): the driver's own staging of small pageable copies is as fast as
    // the ring and needs no thread hand-offs (N=16, 16 cells: 202 against 227 us per collide; 64 cells:
    // 470 against 375, so the ring from there on; profiles/r2_small_bounce_ab.txt)
    if ((size_t)ncells * (size_t)std::max(in_elems, out_elems) * 8 <= (512u << 10)) bounce_in = bounce_out = false;
    if (bounce_in || bounce_out) {
        ensure_bounce(c, chunk);
        return run_host_bounced(c, in, out, in_elems, out_elems, s, max_imag, fn, bounds, two, bounce_in,
                                bounce_out);
    }
    CK(cudaMemsetAsync(c->dFlag, 0, sizeof(int), s));
    if (nchunks == 1) {
        // one chunk has nothing to overlap: copy in, compute and copy out on the caller's stream, with no
        // cross-stream events (a one-cell call is a handful of launches; each hand-off costs microseconds)
        CK(cudaMemcpyAsync(c->dStageIn[0], in, (size_t)ncells * in_elems * 8, cudaMemcpyHostToDevice, s));
        fn(c->dStageIn[0], c->dStageOut[0], ncells, s);
        if (max_imag) CK(cudaMemcpyAsync(max_imag, c->dMaxIm, (size_t)ncells * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(out, c->dStageOut[0], (size_t)ncells * out_elems * 8, cudaMemcpyDeviceToHost, s));
        return check_flag(c, s);
    }
    if (two) {
        CK(cudaEventRecord(c->ev_fork, s));
        CK(cudaStreamWaitEvent(c->comp2, c->ev_fork, 0));
    }
    const int K = c->stage_slots;  // staging slot of chunk i: i % K (compute stream / workspace: i % 2)
    auto h2d = [&](int64_t i) {
        const int slot = (int)(i % K);
        const int64_t c0 = bounds[i], nc = bounds[i + 1] - bounds[i];
        if (i >= K) CK(cudaStreamWaitEvent(c->h2d_stream, c->ev_comp[slot], 0));  // chunk i-K done reading
        CK(cudaMemcpyAsync(c->dStageIn[slot], in + c0 * in_elems, (size_t)nc * in_elems * 8, cudaMemcpyHostToDevice,
                           c->h2d_stream));
        CK(cudaEventRecord(c->ev_h2d[slot], c->h2d_stream));
    };
    h2d(0);
    for (int64_t i = 0; i < nchunks; ++i) {
        const int slot = (int)(i % K);
        const bool odd = (i & 1) && two;
        const int64_t c0 = bounds[i], nc = bounds[i + 1] - bounds[i];
        cudaStream_t cs = odd ? c->comp2 : s;
        CK(cudaStreamWaitEvent(cs, c->ev_h2d[slot], 0));
        if (i >= K) CK(cudaStreamWaitEvent(cs, c->ev_d2h[slot], 0));  // chunk i-K's output left the slot
        {
            WorkspaceSwap ws(c, odd);
            fn(c->dStageIn[slot], c->dStageOut[slot], nc, cs);
            CK(cudaEventRecord(c->ev_comp[slot], cs));
            if (max_imag) CK(cudaMemcpyAsync(max_imag + c0, c->dMaxIm, (size_t)nc * 8, cudaMemcpyDeviceToHost, cs));
        }
        if (i + 1 < nchunks) h2d(i + 1);
        CK(cudaStreamWaitEvent(c->d2h_stream, c->ev_comp[slot], 0));
        CK(cudaMemcpyAsync(out + c0 * out_elems, c->dStageOut[slot], (size_t)nc * out_elems * 8,
                           cudaMemcpyDeviceToHost, c->d2h_stream));
        CK(cudaEventRecord(c->ev_d2h[slot], c->d2h_stream));
    }
    if (two) {
        CK(cudaEventRecord(c->ev_join, c->comp2));
        CK(cudaStreamWaitEvent(s, c->ev_join, 0));
    }
    CK(cudaStreamSynchronize(c->d2h_stream));
    return check_flag(c, s);
}

// Progress counters shared by the bounce pipeline's three host threads.
struct PipeSync {
    std::mutex m;
    std::condition_variable cv;
    int64_t h2d = 0;      // chunks whose H2D is enqueued (ev_h2d recorded)
    int64_t comp = 0;     // chunks whose compute is enqueued (ev_comp recorded)
    int64_t d2h = 0;      // chunks whose D2H is enqueued (ev_d2h recorded)
    int64_t drained = 0;  // chunks copied out to the caller's memory
    bool abort = false;
    std::string err;
    void wait(int64_t PipeSync::*ctr, int64_t v) {
        std::unique_lock<std::mutex> lk(m);
        cv.wait(lk, [&] { return this->*ctr >= v || abort; });
        if (abort) throw CudaError{err.empty() ? std::string("host pipeline aborted") : err};
    }
    void bump(int64_t PipeSync::*ctr) {
        {
            std::lock_guard<std::mutex> g(m);
            ++(this->*ctr);
        }
        cv.notify_all();
    }
    void fail(const std::string& e) {
        {
            std::lock_guard<std::mutex> g(m);
            if (!abort) err = e;
            abort = true;
        }
        cv.notify_all();
    }
};

// The pinned-bounce variant of run_host_pipelined for pageable caller memory.
// Three host threads run the three pipeline legs concurrently, ordered by the
// PipeSync counters and CUDA events:
//   feeder  (chunk i): [pageable in -> pinned slot, in blocks] -> H2D, ev_h2d
//   main    (chunk i): wait ev_h2d; compute on s / comp2; ev_comp
//   drainer (chunk i): wait ev_comp; D2H into the pinned slot in blocks (one
//                      event each); block j -> caller memory while j+1 is in flight
// A direction whose caller memory is pinned skips its bounce copy.
template <typename Fn>
int run_host_bounced(boltz_ctx* c, const double* in, double* out, int in_elems, int out_elems, cudaStream_t s,
                     double* max_imag, Fn& fn, const std::vector<int64_t>& bounds, bool two, bool bounce_in,
                     bool bounce_out) {
    const int64_t nchunks = (int64_t)bounds.size() - 1;
    const int K = c->stage_slots;
    const size_t blk_in = bounce_block();
    auto out_blk = [&](int64_t i) {
        const size_t bytes = (size_t)(bounds[i + 1] - bounds[i]) * out_elems * 8;
        return std::max(bounce_block(), (bytes + boltz_ctx::kBounceBlocks - 1) / boltz_ctx::kBounceBlocks);
    };
    CK(cudaMemsetAsync(c->dFlag, 0, sizeof(int), s));
    if (two) {
        CK(cudaEventRecord(c->ev_fork, s));
        CK(cudaStreamWaitEvent(c->comp2, c->ev_fork, 0));
    }
    // the copy streams must not run ahead of the caller's prior work on `s`
    CK(cudaEventRecord(c->ev_join, s));
    CK(cudaStreamWaitEvent(c->h2d_stream, c->ev_join, 0));
    PipeSync ps;
    auto feeder = [&] {
        try {
            CK(cudaSetDevice(c->device));
            for (int64_t i = 0; i < nchunks; ++i) {
                const int slot = (int)(i % K);
                const int64_t c0 = bounds[i], nc = bounds[i + 1] - bounds[i];
                if (i >= K) {
                    ps.wait(&PipeSync::comp, i - K + 1);  // chunk i-K's ev_comp is recorded
                    CK(cudaStreamWaitEvent(c->h2d_stream, c->ev_comp[slot], 0));  // ... device slot free
                }
                const size_t bytes = (size_t)nc * in_elems * 8;
                if (!bounce_in) {
                    CK(cudaMemcpyAsync(c->dStageIn[slot], in + c0 * in_elems, bytes, cudaMemcpyHostToDevice,
                                       c->h2d_stream));
                } else {
                    if (i >= K) CK(cudaEventSynchronize(c->ev_h2d[slot]));  // pinned slot's last DMA done
                    const char* src = reinterpret_cast<const char*>(in + c0 * in_elems);
                    char* pin = reinterpret_cast<char*>(c->hBounceIn[slot]);
                    char* dst = reinterpret_cast<char*>(c->dStageIn[slot]);
                    for (size_t o = 0; o < bytes; o += blk_in) {
                        const size_t b = std::min(blk_in, bytes - o);
                        host_copy(pin + o, src + o, b);
                        CK(cudaMemcpyAsync(dst + o, pin + o, b, cudaMemcpyHostToDevice, c->h2d_stream));
                    }
                }
                CK(cudaEventRecord(c->ev_h2d[slot], c->h2d_stream));
                ps.bump(&PipeSync::h2d);
            }
        } catch (const CudaError& e) {
            ps.fail(e.msg);
        }
    };
    auto drainer = [&] {
        try {
            CK(cudaSetDevice(c->device));
            for (int64_t i = 0; i < nchunks; ++i) {
                const int slot = (int)(i % K);
                const int64_t c0 = bounds[i], nc = bounds[i + 1] - bounds[i];
                ps.wait(&PipeSync::comp, i + 1);
                CK(cudaStreamWaitEvent(c->d2h_stream, c->ev_comp[slot], 0));
                const size_t bytes = (size_t)nc * out_elems * 8, blk = out_blk(i);
                if (!bounce_out) {
                    CK(cudaMemcpyAsync(out + c0 * out_elems, c->dStageOut[slot], bytes, cudaMemcpyDeviceToHost,
                                       c->d2h_stream));
                    CK(cudaEventRecord(c->ev_d2h[slot], c->d2h_stream));
                    ps.bump(&PipeSync::d2h);
                    ps.bump(&PipeSync::drained);
                    continue;
                }
                char* pin = reinterpret_cast<char*>(c->hBounceOut[slot]);
                const char* src = reinterpret_cast<const char*>(c->dStageOut[slot]);
                int j = 0;
                for (size_t o = 0; o < bytes; o += blk, ++j) {
                    CK(cudaMemcpyAsync(pin + o, src + o, std::min(blk, bytes - o), cudaMemcpyDeviceToHost,
                                       c->d2h_stream));
                    CK(cudaEventRecord(c->ev_blk[slot][j], c->d2h_stream));
                }
                CK(cudaEventRecord(c->ev_d2h[slot], c->d2h_stream));
                ps.bump(&PipeSync::d2h);
                char* dst = reinterpret_cast<char*>(out + c0 * out_elems);
                j = 0;
                for (size_t o = 0; o < bytes; o += blk, ++j) {
                    CK(cudaEventSynchronize(c->ev_blk[slot][j]));
                    host_copy(dst + o, pin + o, std::min(blk, bytes - o));
                }
                if (max_imag) {
                    CK(cudaEventSynchronize(c->ev_comp[slot]));  // the max|Im| copy precedes it on the stream
                    std::memcpy(max_imag + c0, c->hBounceMi[slot], (size_t)nc * 8);
                }
                ps.bump(&PipeSync::drained);
            }
        } catch (const CudaError& e) {
            ps.fail(e.msg);
        }
    };
    static const bool persistent = !(std::getenv("BOLTZ_BOUNCE_PERSIST") && std::atoi(std::getenv("BOLTZ_BOUNCE_PERSIST")) == 0);
    std::thread tf, td;
    bool fed = false, drained = false;
    auto join_legs = [&] {
        if (persistent) {
            if (fed) c->feeder_thread.wait();
            if (drained) c->drainer_thread.wait();
        } else {
            if (tf.joinable()) tf.join();
            if (td.joinable()) td.join();
        }
        fed = drained = false;
    };
    // any other unwinding (e.g. std::bad_alloc on the calling thread) must not
    // leave a leg running on this frame's captures
    struct LegGuard {
        std::function<void()> f;
        ~LegGuard() { f(); }
    } leg_guard{[&] {
        if (fed || drained) {
            ps.fail("host pipeline unwound");
            join_legs();
        }
    }};
    try {
        if (persistent) c->feeder_thread.start(feeder); else tf = std::thread(feeder);
        fed = true;
        if (persistent) c->drainer_thread.start(drainer); else td = std::thread(drainer);
        drained = true;
    } catch (...) {  // a leg may be running: stop it before reporting
        ps.fail("host pipeline: could not start a host thread");
        join_legs();
        throw;
    }
    std::string err;
    try {
        for (int64_t i = 0; i < nchunks; ++i) {
            const int slot = (int)(i % K);
            const bool odd = (i & 1) && two;
            const int64_t c0 = bounds[i], nc = bounds[i + 1] - bounds[i];
            cudaStream_t cs = odd ? c->comp2 : s;
            ps.wait(&PipeSync::h2d, i + 1);
            CK(cudaStreamWaitEvent(cs, c->ev_h2d[slot], 0));
            if (i >= K) {
                ps.wait(&PipeSync::d2h, i - K + 1);  // chunk i-K's output left the device slot
                CK(cudaStreamWaitEvent(cs, c->ev_d2h[slot], 0));
                if (bounce_out && max_imag) ps.wait(&PipeSync::drained, i - K + 1);  // pinned max|Im| slot read
            }
            {
                WorkspaceSwap ws(c, odd);
                fn(c->dStageIn[slot], c->dStageOut[slot], nc, cs);
                if (max_imag)
                    CK(cudaMemcpyAsync(bounce_out ? c->hBounceMi[slot] : max_imag + c0, c->dMaxIm, (size_t)nc * 8,
                                       cudaMemcpyDeviceToHost, cs));
                CK(cudaEventRecord(c->ev_comp[slot], cs));
            }
            ps.bump(&PipeSync::comp);
        }
    } catch (const CudaError& e) {
        err = e.msg;
        ps.fail(e.msg);
    }
    join_legs();
    if (err.empty() && ps.abort) err = ps.err;
    if (!err.empty()) throw CudaError{err};
    if (two) {
        CK(cudaEventRecord(c->ev_join, c->comp2));
        CK(cudaStreamWaitEvent(s, c->ev_join, 0));
    }
    CK(cudaStreamSynchronize(c->d2h_stream));
    return check_flag(c, s);
}

// synchronise `s`, fold timing, report (and clear) the non-finite flag
int check_flag(boltz_ctx* c, cudaStream_t s) {
    CK(cudaMemcpyAsync(c->hFlag, c->dFlag, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (c->timing) collect_timing(c);
    if (*c->hFlag) CK(cudaMemset(c->dFlag, 0, sizeof(int)));
    if (*c->hFlag & 1) {
        set_error("NumericError: non-finite value in the input distribution");
        return BOLTZ_ERR_NUMERIC;
    }
    if (*c->hFlag & 2) {
        set_error("NumericError: non-finite value produced (collision output / RK2 stage)");
        return BOLTZ_ERR_NUMERIC;
    }
    return BOLTZ_OK;
}

template <typename Body>
int api(boltz_ctx* c, Body&& body) {
    int rc = guard_ctx(c);
    if (rc) return rc;
    try {
        return body();
    } catch (const CudaError& e) {
        set_error(e.msg);
        return BOLTZ_ERR_CUDA;
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed");
        return BOLTZ_ERR_CUDA;
    } catch (const std::exception& e) {  // e.g. std::system_error from the host pipeline's threads
        set_error(std::string("host runtime error: ") + e.what());
        return BOLTZ_ERR_CUDA;
    }
}

}  // namespace

namespace {
int create_context(int n, double L, double lambda, double beta, double r0, int panels, const double* G_host,
                   int device, boltz_ctx** out, bool with_table = true);

// the collision entry points need the weight table (boltz_create_transform has none)
int need_table(const boltz_ctx* c) {
    if (c->dH) return BOLTZ_OK;
    set_error("this context has no weight table (boltz_create_transform): transforms only");
    return BOLTZ_ERR_CONFIG;
}
}

extern "C" {

const char* boltz_last_error(void) { return g_err.c_str(); }

const char* boltz_build_info(void) {
    return "boltz_cuda sm_100a; N in {4,6,8,12,16,24,32}; conv: pair-symmetric folded table, lane=cell group layout";
}

int boltz_create(int n, double L, double lambda, double beta, double r0, const double* G_host, int device,
                 boltz_ctx** out) {
    if (!out) {
        set_error("boltz_create: out is null");
        return BOLTZ_ERR_CONFIG;
    }
    *out = nullptr;
    if (n < 4 || n % 2 != 0) {
        set_error("velocity grid: N must be even and >= 4, got " + std::to_string(n));
        return BOLTZ_ERR_CONFIG;
    }
    if (!(L > 0.0)) {
        set_error("velocity grid: L must be positive, got " + std::to_string(L));
        return BOLTZ_ERR_CONFIG;
    }
    if (!supported_n(n)) {
        set_error("boltz_create: N=" + std::to_string(n) + " has no compiled kernel (supported 4,6,8,12,16,24,32)");
        return BOLTZ_ERR_CONFIG;
    }
    if (!(lambda >= 0.0 && lambda <= 1.0) || !(beta > 0.0 && beta <= 1.0) || !(r0 > 0.0)) {
        set_error("kernel spec: need 0<=lambda<=1, 0<beta<=1, r0>0");
        return BOLTZ_ERR_CONFIG;
    }
    if (!G_host) {
        set_error("boltz_create: weight table is null");
        return BOLTZ_ERR_CONFIG;
    }
    return create_context(n, L, lambda, beta, r0, 64, G_host, device, out);
}

int boltz_create_generated(int n, double L, double lambda, double beta, double r0, int panels, int device,
                           boltz_ctx** out) {
    if (!out) {
        set_error("boltz_create_generated: out is null");
        return BOLTZ_ERR_CONFIG;
    }
    *out = nullptr;
    if (n < 4 || n % 2 != 0 || !(L > 0.0)) {
        set_error("velocity grid: N must be even and >= 4 and L > 0");
        return BOLTZ_ERR_CONFIG;
    }
    if (!supported_n(n)) {
        set_error("boltz_create_generated: N=" + std::to_string(n) + " has no compiled kernel");
        return BOLTZ_ERR_CONFIG;
    }
    if (!(lambda >= 0.0 && lambda <= 1.0) || !(beta > 0.0 && beta <= 1.0) || !(r0 > 0.0) || panels < 1) {
        set_error("kernel spec: need 0<=lambda<=1, 0<beta<=1, r0>0, panels>=1");
        return BOLTZ_ERR_CONFIG;
    }
    return create_context(n, L, lambda, beta, r0, panels, nullptr, device, out);
}

int boltz_create_transform(int n, double L, int device, boltz_ctx** out) {
    if (!out) {
        set_error("boltz_create_transform: out is null");
        return BOLTZ_ERR_CONFIG;
    }
    *out = nullptr;
    if (n < 4 || n % 2 != 0 || !(L > 0.0)) {
        set_error("velocity grid: N must be even and >= 4 and L > 0");
        return BOLTZ_ERR_CONFIG;
    }
    if (!supported_n(n)) {
        set_error("boltz_create_transform: N=" + std::to_string(n) + " has no compiled kernel");
        return BOLTZ_ERR_CONFIG;
    }
    return create_context(n, L, 1.0, 1.0, L, 64, nullptr, device, out, false);
}

}  // extern "C"

namespace {
int create_context(int n, double L, double lambda, double beta, double r0, int panels, const double* G_host,
                   int device, boltz_ctx** out, bool with_table) {
    boltz_ctx* c = new boltz_ctx();
    c->n = n; c->L = L; c->lambda = lambda; c->beta = beta; c->r0 = r0; c->device = device; c->panels = panels;
    if (const char* e = std::getenv("BOLTZ_LINE_CPB"))  // tuning: cells per CTA of the line kernels, device calls
        c->line_cpb = std::atoi(e) == 1 ? 1 : 2;
    if (const char* e = std::getenv("BOLTZ_STAGE_SLOTS"))  // tuning
        c->stage_slots = std::min(boltz_ctx::kMaxStageSlots, std::max(2, std::atoi(e)));
    try {
        CK(cudaSetDevice(device));
        CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
        CK(cudaMalloc(&c->dFlag, sizeof(int)));
        CK(cudaMemset(c->dFlag, 0, sizeof(int)));
        CK(cudaStreamCreateWithFlags(&c->h2d_stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->comp2, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
        for (int b = 0; b < boltz_ctx::kMaxStageSlots; ++b) {
            CK(cudaEventCreateWithFlags(&c->ev_h2d[b], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c->ev_comp[b], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&c->ev_d2h[b], cudaEventDisableTiming));
        }
        CK(cudaMallocHost(&c->hFlag, sizeof(int)));
        fill_twiddles();
        build_projection(c);
        if (with_table) build_table(c, G_host);
    } catch (const CudaError& e) {
        set_error(e.msg);
        boltz_destroy(c);
        return BOLTZ_ERR_CUDA;
    } catch (const std::exception& e) {  // host allocation of the table layout
        set_error(std::string("boltz_create: ") + e.what());
        boltz_destroy(c);
        return BOLTZ_ERR_CUDA;
    }
    *out = c;
    return BOLTZ_OK;
}
}  // namespace

extern "C" {

int boltz_destroy(boltz_ctx* c) {
    if (!c) return BOLTZ_OK;
    cudaSetDevice(c->device);
    cudaFree(c->dH); cudaFree(c->dEnt); cudaFree(c->dRowStart);
    cudaFree(c->dMH); cudaFree(c->dMEnt); cudaFree(c->dItems); for (int* l : c->dListK) cudaFree(l);
    cudaFree(c->dA); cudaFree(c->dB); cudaFree(c->dFs);
    cudaFree(c->dMaxIm); cudaFree(c->dFlag);
    cudaFree(c->dA2); cudaFree(c->dB2); cudaFree(c->dFs2); cudaFree(c->dMaxIm2);
    cudaFree(c->dSeg); cudaFree(c->dSeg2); cudaFree(c->dCell); cudaFree(c->dCell2);
    for (void* p : c->retired) cudaFree(p);
    if (c->comp2) cudaStreamDestroy(c->comp2);
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_join) cudaEventDestroy(c->ev_join);
    for (int b = 0; b < boltz_ctx::kMaxStageSlots; ++b) {
        cudaFree(c->dStageIn[b]);
        cudaFree(c->dStageOut[b]);
        if (c->ev_h2d[b]) cudaEventDestroy(c->ev_h2d[b]);
        if (c->ev_comp[b]) cudaEventDestroy(c->ev_comp[b]);
        if (c->ev_d2h[b]) cudaEventDestroy(c->ev_d2h[b]);
    }
    if (c->h2d_stream) cudaStreamDestroy(c->h2d_stream);
    if (c->d2h_stream) cudaStreamDestroy(c->d2h_stream);
    if (c->hFlag) cudaFreeHost(c->hFlag);
    for (int b = 0; b < boltz_ctx::kMaxStageSlots; ++b) {
        if (c->hBounceIn[b]) cudaFreeHost(c->hBounceIn[b]);
        if (c->hBounceOut[b]) cudaFreeHost(c->hBounceOut[b]);
        if (c->hBounceMi[b]) cudaFreeHost(c->hBounceMi[b]);
        for (cudaEvent_t e : c->ev_blk[b])
            if (e) cudaEventDestroy(e);
    }
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    delete c;
    return BOLTZ_OK;
}

int boltz_memory_bytes(const boltz_ctx* c, int64_t* table_bytes, int64_t* workspace_bytes) {
    if (!c) return BOLTZ_ERR_CONFIG;
    if (table_bytes) *table_bytes = c->table_bytes;
    if (workspace_bytes) *workspace_bytes = c->ws_bytes;
    return BOLTZ_OK;
}

int boltz_forward_batch(boltz_ctx* c, const double* f, double* fhat, int64_t ncells, int mem, void* stream) {
    return api(c, [&] {
        const int64_t n3 = n3_of(c);
        return run_chunked(c, f, fhat, ncells, (int)n3, (int)(2 * n3), mem, stream, nullptr,
                           [&](const double* in, double* out, int64_t nc, cudaStream_t s) {
                               dispatch(c->n, [&](auto L) {
                                   using Lx = decltype(L);
                                   Lx::forward(c, in, nc, s);
                                   Lx::unpack_complex(c, c->dA, out, nc, 0, s);
                               });
                           });
    });
}

int boltz_inverse_batch(boltz_ctx* c, const double* g, double* f, double* max_imag, int64_t ncells, int mem,
                        void* stream) {
    return api(c, [&] {
        const int64_t n3 = n3_of(c);
        return run_chunked(c, g, f, ncells, (int)(2 * n3), (int)n3, mem, stream, max_imag,
                           [&](const double* in, double* out, int64_t nc, cudaStream_t s) {
                               dispatch(c->n, [&](auto L) {
                                   using Lx = decltype(L);
                                   Lx::pack_complex(c, in, c->dB, nc, 1, s);
                                   Lx::inverse(c, nc, s);
                                   Lx::unpack_real(c, reinterpret_cast<const double*>(c->dA), out, nc, s);
                               });
                           });
    });
}

int boltz_qhat_batch(boltz_ctx* c, const double* fhat, double* qhat, int64_t ncells, int mem, void* stream) {
    return api(c, [&] {
        if (int rc = need_table(c)) return rc;
        const int64_t n3 = n3_of(c);
        return run_chunked(c, fhat, qhat, ncells, (int)(2 * n3), (int)(2 * n3), mem, stream, nullptr,
                           [&](const double* in, double* out, int64_t nc, cudaStream_t s) {
                               dispatch(c->n, [&](auto L) {
                                   using Lx = decltype(L);
                                   Lx::pack_complex(c, in, c->dA, nc, 0, s);
                                   Lx::conv(c, nc, s);  // a caller's fhat: plain schedule
                                   Lx::unpack_complex(c, c->dB, out, nc, 1, s);
                               });
                           });
    });
}

int boltz_conserve_batch(boltz_ctx* c, const double* q_raw, double* q, int64_t ncells, int mem, void* stream) {
    return api(c, [&] {
        const int64_t n3 = n3_of(c);
        return run_chunked(c, q_raw, q, ncells, (int)n3, (int)n3, mem, stream, nullptr,
                           [&](const double* in, double* out, int64_t nc, cudaStream_t s) {
                               dispatch(c->n, [&](auto L) {
                                   using Lx = decltype(L);
                                   Lx::pack_real(c, in, reinterpret_cast<double*>(c->dA), nc, s);
                                   Lx::project(c, nullptr, out, nc, 1.0, s);
                               });
                           });
    });
}

int boltz_collide_batch(boltz_ctx* c, const double* f, double* q, int64_t ncells, double inv_eps, double* max_imag,
                        int mem, void* stream) {
    return api(c, [&] {
        if (int rc = need_table(c)) return rc;
        const int64_t n3 = n3_of(c);
        return run_chunked(c, f, q, ncells, (int)n3, (int)n3, mem, stream, max_imag,
                           [&](const double* in, double* out, int64_t nc, cudaStream_t s) {
                               dispatch(c->n, [&](auto L) {
                                   using Lx = decltype(L);
                                   Lx::forward(c, in, nc, s);
                                   Lx::conv(c, nc, s, true);  // fhat of a real f: mirror schedule
                                   Lx::inverse_project(c, nullptr, out, nc, inv_eps, s);
                               });
                           });
    });
}

int boltz_rk2_batch(boltz_ctx* c, double* f, int64_t ncells, double dt, double inv_eps, int mem, void* stream) {
    return api(c, [&] {
        if (int rc = need_table(c)) return rc;
        const int64_t n3 = n3_of(c);
        return run_chunked(c, f, f, ncells, (int)n3, (int)n3, mem, stream, nullptr,
                           [&](const double* in, double* out, int64_t nc, cudaStream_t s) {
                               // host staging: in = dIn, out = dOut; copy base through
                               if (in != out) CK(cudaMemcpyAsync(out, in, (size_t)nc * n3 * 8,
                                                                 cudaMemcpyDeviceToDevice, s));
                               dispatch(c->n, [&](auto L) {
                                   using Lx = decltype(L);
                                   // stage 1: f* = f + dt/2 * collide(f)
                                   Lx::forward(c, out, nc, s);
                                   Lx::conv(c, nc, s, true);  // fhat of a real f: mirror schedule
                                   // stage 2: f <- f + dt * collide(f*), f* handed over as fhat(f*)
                                   Lx::inverse_project_forward(c, out, c->dFs, nc, 0.5 * dt * inv_eps, s);
                                   Lx::conv(c, nc, s, true);  // fhat of a real f: mirror schedule
                                   Lx::inverse_project(c, out, out, nc, dt * inv_eps, s);
                               });
                           });
    });
}

int boltz_transport_step(boltz_ctx* c, const double* field, const double* base, double alpha, double* out,
                         int64_t ncl, const double* x_ext, const double* dx_ext, double dt, int wall_left,
                         int wall_right, void* stream) {
    return api(c, [&] {
        if (ncl < 1 || !field || !out || !x_ext || !dx_ext || out == field || (base && out == base)) {
            set_error("transport_step: invalid arguments (out must not alias field/base)");
            return BOLTZ_ERR_CONFIG;
        }
        cudaStream_t s = (cudaStream_t)stream;  // NULL = the CUDA default stream
        {
            Timed t_(c, KIND_TRANSPORT, s);
            launch_transport(c->n, field, base, base ? alpha : 0.0, out, ncl, x_ext, dx_ext, dt, wall_left,
                             wall_right, c->pc.dv, s);
        }
        CK(cudaGetLastError());
        if (c->async_mode) return BOLTZ_OK;
        CK(cudaStreamSynchronize(s));
        if (c->timing) collect_timing(c);
        return BOLTZ_OK;
    });
}

int boltz_transport_step_range(boltz_ctx* c, const double* field, const double* base, double alpha, double* out,
                               int64_t ncl, const double* x_ext, const double* dx_ext, double dt, int wall_left,
                               int wall_right, int64_t c_begin, int64_t c_end, void* stream) {
    return api(c, [&] {
        if (ncl < 1 || !field || !out || !x_ext || !dx_ext || out == field || (base && out == base) || c_begin < 2 ||
            c_end > ncl + 2 || c_begin > c_end) {
            set_error("transport_step_range: invalid arguments (need 2 <= c_begin <= c_end <= ncl + 2; out must not "
                      "alias field/base)");
            return BOLTZ_ERR_CONFIG;
        }
        cudaStream_t s = (cudaStream_t)stream;
        {
            Timed t_(c, KIND_TRANSPORT, s);
            launch_transport(c->n, field, base, base ? alpha : 0.0, out, ncl, x_ext, dx_ext, dt, wall_left,
                             wall_right, c->pc.dv, s, 0, nullptr, nullptr, c_begin, c_end);
        }
        CK(cudaGetLastError());
        if (c->async_mode) return BOLTZ_OK;
        CK(cudaStreamSynchronize(s));
        if (c->timing) collect_timing(c);
        return BOLTZ_OK;
    });
}

int boltz_transport_step_peer(boltz_ctx* c, const double* field, const double* base, double alpha, double* out,
                              int64_t ncl, const double* x_ext, const double* dx_ext, double dt, int wall_left,
                              int wall_right, double* left_dst, double* right_dst, void* stream) {
    return api(c, [&] {
        if (ncl < 2 || !field || !out || !x_ext || !dx_ext || out == field || (base && out == base)) {
            set_error("transport_step_peer: invalid arguments (out must not alias field/base, ncl >= 2)");
            return BOLTZ_ERR_CONFIG;
        }
        cudaStream_t s = (cudaStream_t)stream;
        {
            Timed t_(c, KIND_TRANSPORT, s);
            launch_transport(c->n, field, base, base ? alpha : 0.0, out, ncl, x_ext, dx_ext, dt, wall_left,
                             wall_right, c->pc.dv, s, 1, left_dst, right_dst);
        }
        CK(cudaGetLastError());
        if (c->async_mode) return BOLTZ_OK;
        CK(cudaStreamSynchronize(s));
        if (c->timing) collect_timing(c);
        return BOLTZ_OK;
    });
}

int boltz_store_edges(boltz_ctx* c, const double* interior, int64_t ncells, double* left_dst, double* right_dst,
                      void* stream) {
    return api(c, [&] {
        if (ncells < 2 || !interior) {
            set_error("store_edges: need >= 2 interior cells");
            return BOLTZ_ERR_CONFIG;
        }
        cudaStream_t s = (cudaStream_t)stream;
        {
            Timed t_(c, KIND_TRANSPORT, s);
            launch_store_edges(c->n, interior, ncells, left_dst, right_dst, s);
        }
        CK(cudaGetLastError());
        if (c->async_mode) return BOLTZ_OK;
        CK(cudaStreamSynchronize(s));
        return BOLTZ_OK;
    });
}

int boltz_end_flux(boltz_ctx* c, const double* field, int64_t ncl, const double* x_ext, const double* dx_ext,
                   int wall_left, int wall_right, double coef, double* acc5, void* stream) {
    return api(c, [&] {
        if (ncl < 1 || !field || !x_ext || !dx_ext || !acc5) {
            set_error("end_flux: invalid arguments");
            return BOLTZ_ERR_CONFIG;
        }
        cudaStream_t s = (cudaStream_t)stream;  // NULL = the CUDA default stream
        {
            Timed t_(c, KIND_TRANSPORT, s);
            launch_end_flux(c->n, field, ncl, x_ext, dx_ext, wall_left, wall_right, c->pc.dv, coef, acc5, s);
        }
        CK(cudaGetLastError());
        if (c->async_mode) return BOLTZ_OK;
        CK(cudaStreamSynchronize(s));
        return BOLTZ_OK;
    });
}

int boltz_fill_boundary(boltz_ctx* c, double* field, int64_t ncl, const double* x_ext, int side, int kind, double Tw,
                        const double* Vw_host3, double* sigma_w, void* stream) {
    return api(c, [&] {
        if (ncl < 2 || !field || !x_ext || (side != 0 && side != 1) || kind < 0 || kind > 2) {
            set_error("fill_boundary: invalid arguments (need >= 2 interior cells)");
            return BOLTZ_ERR_CONFIG;
        }
        if (kind != 0 && !(Tw > 0.0)) {
            set_error("fill_boundary: wall temperature must be positive");
            return BOLTZ_ERR_CONFIG;
        }
        cudaStream_t s = (cudaStream_t)stream;  // NULL = the CUDA default stream
        note_capture(c, s);
        double vw[3] = {0, 0, 0};
        if (Vw_host3) std::memcpy(vw, Vw_host3, sizeof vw);
        double* dsig = reinterpret_cast<double*>(c->dMaxIm);
        if (!dsig) {
            ensure_workspace(c, kLanes);
            dsig = reinterpret_cast<double*>(c->dMaxIm);
        }
        {
            Timed t_(c, KIND_TRANSPORT, s);
            launch_fill_boundary(c->n, field, ncl, x_ext, side, kind, Tw, vw[0], vw[1], vw[2], c->pc.dv, dsig, s);
        }
        CK(cudaGetLastError());
        if (c->async_mode) return BOLTZ_OK;  // sigma_w stays on the device (not reported)
        double hs = 0.0;
        CK(cudaMemcpyAsync(&hs, dsig, sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (c->timing) collect_timing(c);
        if (sigma_w) *sigma_w = hs;
        return BOLTZ_OK;
    });
}

int boltz_moments_batch(boltz_ctx* c, const double* f, double* out, int64_t ncells, int mem, void* stream) {
    return api(c, [&] {
        const int64_t n3 = n3_of(c);
        return run_chunked(c, f, out, ncells, (int)n3, 7, mem, stream, nullptr,
                           [&](const double* in, double* o, int64_t nc, cudaStream_t s) {
                               Timed t_(c, KIND_LAYOUT, s);
                               launch_moments(c->n, in, o, nc, c->pc.dv, s);
                               CK(cudaGetLastError());
                           });
    });
}

int boltz_marginal_batch(boltz_ctx* c, const double* f, double* g, int64_t ncells, int mem, void* stream) {
    return api(c, [&] {
        const int64_t n3 = n3_of(c);
        return run_chunked(c, f, g, ncells, (int)n3, c->n, mem, stream, nullptr,
                           [&](const double* in, double* o, int64_t nc, cudaStream_t s) {
                               Timed t_(c, KIND_LAYOUT, s);
                               launch_marginal(c->n, in, o, nc, c->pc.dv, s);
                               CK(cudaGetLastError());
                           });
    });
}

const char* boltz_conv_kernel(const boltz_ctx* c) {
    if (!c) return "";
    if (c->schedule == kScheduleAuto && c->n <= 16) return "auto: k_conv_cell / k_conv_seg / mirror by batch size";
    if (c->schedule == kScheduleCell && c->n <= 16) return "k_conv_cell + k_cell_gather";
    if (c->schedule > 0 && c->schedule < kScheduleCell && c->n <= 16) return "k_conv_seg + k_conv_seg_reduce";
    if (c->mirror) {
        if (c->mirror2) return "k_conv_mirror2";
        if (mirror_pipe_n(c->n)) return "k_conv_mirror";
        return c->n == 32 ? (kcsf_n(32) ? "k_conv_kcsm (phase 0 with the REST fold, phase 2)" : "k_conv_kcsm (phases 0, 2) + k_conv_kcsr") : "k_conv_kcsm";
    }
    return conv_kernel_for(c->n) == 1 ? "k_conv_pipe" : "k_conv_kcs";
}

int boltz_schedule_terms(boltz_ctx* c, int64_t* plain, int64_t* mirror) {
    if (!c) return BOLTZ_ERR_CONFIG;
    if (plain) *plain = c->terms_plain;
    if (mirror) *mirror = c->mirror ? c->terms_mirror : 0;
    return BOLTZ_OK;
}

int boltz_set_schedule(boltz_ctx* c, int schedule) {
    if (!c || schedule < 0 || schedule > kScheduleAuto) {
        set_error("set_schedule: 0 (throughput), 1..4 (latency: 4 x schedule segments per row), 5 (cell) or 6 (auto)");
        return BOLTZ_ERR_CONFIG;
    }
    c->schedule = schedule;
    return BOLTZ_OK;
}

int boltz_set_async(boltz_ctx* c, int enable) {
    if (!c) return BOLTZ_ERR_CONFIG;
    c->async_mode = enable != 0;
    return BOLTZ_OK;
}

int boltz_sync(boltz_ctx* c, void* stream) {
    return api(c, [&] { return check_flag(c, (cudaStream_t)stream); });
}

int boltz_set_timing(boltz_ctx* c, int enable) {
    if (!c) return BOLTZ_ERR_CONFIG;
    c->timing = enable != 0;
    return BOLTZ_OK;
}

int boltz_get_timing(boltz_ctx* c, double* ms, int64_t* launches, int nkinds, int reset) {
    if (!c || nkinds < 0) return BOLTZ_ERR_CONFIG;
    for (int k = 0; k < nkinds && k < kKinds; ++k) {
        if (ms) ms[k] = c->ms[k];
        if (launches) launches[k] = c->launches[k];
    }
    if (reset)
        for (int k = 0; k < kKinds; ++k) {
            c->ms[k] = 0.0;
            c->launches[k] = 0;
        }
    return BOLTZ_OK;
}

int boltz_fp64_peak(int device, double seconds, double* tflops) {
    try {
        CK(cudaSetDevice(device));
        *tflops = fp64_peak_probe(seconds);
        return BOLTZ_OK;
    } catch (const CudaError& e) {
        set_error(e.msg);
        return BOLTZ_ERR_CUDA;
    }
}

}  // extern "C"
