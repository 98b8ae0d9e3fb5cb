/*
 * boltz_cuda.h -- C ABI of the B200 (sm_100a) collision path.
 *
 * Drop-in boundary for the reference's per-cell collision step (SURVEY.md
 * §8b).  Each entry point replaces one reference operation, batched over
 * cells; no torch or C++ types cross the boundary, no exceptions escape.
 *
 *   reference operation                                   | entry point
 *   ------------------------------------------------------+-------------------------------
 *   SpectralTransform(grid)           fourier.hpp:31       | boltz_create (+ table upload)
 *   ~SpectralTransform                fourier.hpp:32       | boltz_destroy
 *   SpectralTransform::forward        fourier.hpp:36       | boltz_forward_batch
 *   SpectralTransform::inverse        fourier.hpp:38-41    | boltz_inverse_batch
 *   evaluate_qhat                     SPEC.md:186-194      | boltz_qhat_batch
 *   conserve                          SPEC.md:204-212      | boltz_conserve_batch
 *   collide                           SPEC.md:195-203      | boltz_collide_batch
 *   collision_rk2                     SPEC.md:383-391      | boltz_rk2_batch
 *   generate_table                    SPEC.md:126-134      | boltz_generate_table (host)
 *   save_table / load_table           SPEC.md:135-143      | boltz_save_table / boltz_load_table
 *   transport_step (+ ghost fill)     SPEC.md:342-350      | boltz_transport_step
 *   boltz::Error{category}            errors.hpp:8-35      | return codes + boltz_last_error
 *
 * Layouts at the boundary are the reference's: a batch of `ncells` cells is
 * `ncells` consecutive N^3 blocks, flat index (i1*N+i2)*N+i3
 * (velocity_grid.hpp:30-32); complex arrays are interleaved (re, im) doubles
 * (std::complex<double>, fourier.hpp:36).  The weight table is the dense
 * zeta-major N^6 array G[k][m].
 *
 * `mem`: BOLTZ_MEM_HOST (pointers are host memory; the call copies in/out
 * and is synchronous) or BOLTZ_MEM_DEVICE (pointers are device memory on the
 * context's device; the call is ordered on `stream` and synchronises it
 * before returning so that numeric errors can be reported).  `stream` may be
 * NULL (the CUDA default stream), as in any CUDA API.
 *
 * Threading mirrors SpectralTransform (fourier.hpp:24-25): a context is not
 * thread-safe; distinct contexts may be used concurrently.
 */
#ifndef BOLTZ_CUDA_H
#define BOLTZ_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* return codes: 0 ok; 2/3/4 mirror boltz::ErrorCategory (errors.hpp:8-13) */
#define BOLTZ_OK 0
#define BOLTZ_ERR_CONFIG 2
#define BOLTZ_ERR_IO 3
#define BOLTZ_ERR_NUMERIC 4
#define BOLTZ_ERR_CUDA 5 /* CUDA / NCCL failure (new; no reference counterpart) */

#define BOLTZ_MEM_HOST 0
#define BOLTZ_MEM_DEVICE 1

typedef struct boltz_ctx boltz_ctx;

/* Thread-local message of the last failing call ("" if none). */
const char* boltz_last_error(void);

/* Library build information (compute capability, supported N list). */
const char* boltz_build_info(void);

/*
 * Create a context on `device` for the grid (n, L) (VelocityGrid::create,
 * velocity_grid.cpp:11-32: n even >= 4, L > 0) and kernel (lambda, beta, r0)
 * (KernelSpec).  `G_host` is the caller's dense zeta-major
 * table (n^6 doubles); it is COPIED (and re-laid out) into device memory and
 * may be freed after the call.  Errors: 2 for an invalid grid/kernel or an
 * unsupported n, 5 for CUDA failures (e.g. out of device memory).
 */
int boltz_create(int n, double L, double lambda, double beta, double r0, const double* G_host, int device,
                 boltz_ctx** out);
int boltz_destroy(boltz_ctx* ctx);

/*
 * As boltz_create, but the weight table is evaluated on the device (same
 * closed forms / Gauss-Legendre quadrature with `panels` panels as
 * boltz_generate_table) straight into the folded layout -- no host N^6 table
 * (the reference generates on the host).
 */
int boltz_create_generated(int n, double L, double lambda, double beta, double r0, int panels, int device,
                           boltz_ctx** out);

/* Device bytes held by the context (folded table + workspace). */
/* A transforms-only context (no weight table): forward / inverse / conserve /
 * moments / marginal / transport work, collision calls return
 * BOLTZ_ERR_CONFIG.  Backs the reference-typed boltz::SpectralTransform
 * (fourier.hpp:28-52) of paper_1301_4195_b200/shim/fourier_cuda.cpp. */
int boltz_create_transform(int n, double L, int device, boltz_ctx** out);

int boltz_memory_bytes(const boltz_ctx* ctx, int64_t* table_bytes, int64_t* workspace_bytes);

/* forward: f (ncells x N^3 real) -> fhat (ncells x N^3 complex) */
int boltz_forward_batch(boltz_ctx* ctx, const double* f, double* fhat, int64_t ncells, int mem, void* stream);

/* inverse: g (complex) -> f (real); max_imag (ncells doubles, nullable) */
int boltz_inverse_batch(boltz_ctx* ctx, const double* g, double* f, double* max_imag, int64_t ncells, int mem,
                        void* stream);

/* evaluate_qhat: fhat (complex) -> qhat (complex), raw K2 for parity tests */
int boltz_qhat_batch(boltz_ctx* ctx, const double* fhat, double* qhat, int64_t ncells, int mem, void* stream);

/* conserve: q_raw (real) -> q (real) */
int boltz_conserve_batch(boltz_ctx* ctx, const double* q_raw, double* q, int64_t ncells, int mem, void* stream);

/*
 * collide: q = (1/eps) P_N(inverse(evaluate_qhat(forward(f)))) per cell.
 * inv_eps = 1/epsilon.  max_imag (ncells, nullable): inverse-transform
 * imaginary residue (fourier.hpp:38-41).  Non-finite f -> 4.
 */
int boltz_collide_batch(boltz_ctx* ctx, const double* f, double* q, int64_t ncells, double inv_eps,
                        double* max_imag, int mem, void* stream);

/*
 * collision_rk2 in place: f* = f + dt/2 collide(f); f <- f + dt collide(f*).
 * Non-finite input or stage -> 4.
 */
int boltz_rk2_batch(boltz_ctx* ctx, double* f, int64_t ncells, double dt, double inv_eps, int mem, void* stream);

/*
 * transport_step on a device field of (ncl + 4) cells x
 * N^3 (2 ghost cells per side) whose ghosts are already filled
 * (halo exchange / boltz_fill_boundary).  x_ext, dx_ext: DEVICE arrays of the
 * ncl+4 cell centres/widths.  wall_left/right: zero slope at a wall
 * (SPEC.md:336,359).  `out` (device, same shape, not aliasing field/base)
 * receives alpha*base + (1-alpha)*step(field) on interior cells (base NULL:
 * the plain step), its ghost cells are copied through.  base/alpha fuse the
 * second stage of the SSP-RK2 transport sub-step.
 */
int boltz_transport_step(boltz_ctx* ctx, const double* field, const double* base, double alpha, double* out,
                         int64_t ncl, const double* x_ext, const double* dx_ext, double dt, int wall_left,
                         int wall_right, void* stream);

/* transport_step on the interior rows [c_begin, c_end) only (2 <= c_begin <=
 * c_end <= ncl + 2; field rows are cells, ghosts at 0, 1, ncl + 2, ncl + 3).
 * Rows c_begin >= 4 and c_end <= ncl read no ghost row, so they can run while
 * the halo exchange is in flight; the left ghost rows are copied through iff
 * c_begin == 2, the right ones iff c_end == ncl + 2.  Bitwise the rows of the
 * whole-interior call (halo/compute overlap). */
int boltz_transport_step_range(boltz_ctx* ctx, const double* field, const double* base, double alpha, double* out,
                               int64_t ncl, const double* x_ext, const double* dx_ext, double dt, int wall_left,
                               int wall_right, int64_t c_begin, int64_t c_end, void* stream);

/*
 * The halo exchange fused into the transport step (B200 peer memory; no
 * reference counterpart -- it replaces transport_step + halo_exchange,
 * SPEC.md:342-350,446-453).  Same step as boltz_transport_step, plus: the
 * updated cells 2,3 are also stored at left_dst (the left rank's output field
 * + (ncl_left + 2) * N^3, i.e. its right ghosts) and cells ncl, ncl+1 at
 * right_dst (the right rank's output field, i.e. its left ghosts 0,1); null =
 * no neighbour.  This rank's own ghost rows of `out` are not written (its
 * neighbours and boltz_fill_boundary own them).  Pointers are device or peer
 * (cudaDeviceEnablePeerAccess / IPC) addresses.  The caller orders each step
 * after the neighbours' previous step (events) -- see include/boltz_solver.hpp.
 */
int boltz_transport_step_peer(boltz_ctx* ctx, const double* field, const double* base, double alpha, double* out,
                              int64_t ncl, const double* x_ext, const double* dx_ext, double dt, int wall_left,
                              int wall_right, double* left_dst, double* right_dst, void* stream);
/* the collision step's half of the fused exchange: interior cells 0,1 ->
 * left_dst, ncells-2, ncells-1 -> right_dst (addressing as above) */
int boltz_store_edges(boltz_ctx* ctx, const double* interior, int64_t ncells, double* left_dst, double* right_dst,
                      void* stream);

/*
 * Boundary-flux ledger (reference SPEC.md:403 "conservation ledger ... vs
 * wall-flux integral"; RunRecord): acc5[a] += coef * (F_a(right face) -
 * F_a(left face)) for the 5 collision invariants (mass, momentum 1-3, energy
 * |v|^2/2), through the faces of the first and last interior cells of this
 * rank's field -- the exact face values boltz_transport_step uses.  acc5 is a
 * DEVICE array of 5 doubles.  For one SSP-RK2 transport sub-step of size h,
 * calling it with coef = h/2 before each of the two FV stages makes
 * sum_ranks ledger(t) + acc constant to round-off.
 */
int boltz_end_flux(boltz_ctx* ctx, const double* field, int64_t ncl, const double* x_ext, const double* dx_ext,
                   int wall_left, int wall_right, double coef, double* acc5, void* stream);

/*
 * Ghost fill at a physical end (side 0 = left, 1 = right) of a device field:
 * kind 0 = linear extrapolation, kind 1 = diffuse wall with
 * T_w, V_w (sigma_w from the continuum half-range integral,
 * so the lattice mass flux through the wall is only balanced to O(dv^2)),
 * kind 2 = extension: the same wall with sigma_w from the discrete flux
 * balance (lattice influx == outflux; zero net wall mass flux to round-off).
 * x_ext is a DEVICE array.  sigma_w (host double, nullable) receives the
 * wall's re-emission factor.
 */
int boltz_fill_boundary(boltz_ctx* ctx, double* field, int64_t ncl, const double* x_ext, int side, int kind,
                        double Tw, const double* Vw_host3, double* sigma_w, void* stream);

/*
 * compute_moments per cell: out[c*7 + {0..6}] = rho,
 * rho V1, rho V2, rho V3, rho e, T, H (H = sum_{f>0} f log f w; R = 1).
 */
int boltz_moments_batch(boltz_ctx* ctx, const double* f, double* out, int64_t ncells, int mem, void* stream);

/*
 * marginal_distribution (reference SPEC.md cli_io module, "[OP]
 * marginal_distribution"; the Figure-4 output): g[c*N + i] = sum over v2, v3
 * of f w2 w3 at v1 = dv (i - N/2), w = trapezoid coefficient x dv.
 */
int boltz_marginal_batch(boltz_ctx* ctx, const double* f, double* g, int64_t ncells, int mem, void* stream);

/*
 * Asynchronous mode (no reference counterpart): with
 * enable != 0, device-pointer calls return as soon as their work is queued on
 * the stream (no synchronisation, so a whole Strang step can be captured in a
 * CUDA graph); non-finite detections accumulate and are reported -- and the
 * stream synchronised -- by boltz_sync.  fill_boundary does not report
 * sigma_w in this mode.  Host-pointer calls stay synchronous.
 */
/*
 * K2 schedule (no reference counterpart): 0 = throughput (default; one warp per
 * output row, or per mirror row pair, and 32-cell group), s = 1..4 = latency
 * (each row's entry list in 4s fixed segments on 4s warps + an ordered
 * reduction; small batches, N <= 16; other N keep the throughput schedule),
 * 5 = cell (lane = output k3, one CTA per (output row, cell), the cell's
 * f-hat in shared memory: one or a few cells, N <= 16; conv.cuh k_conv_cell).
 * 6 = auto: chosen per call from the batch size at N <= 16 (<= 4 cells: cell;
 * <= 64: latency with 8 segments; <= 256: latency with 4; else throughput) --
 * for callers that, like the reference's strang_step, pass
 * one or a few cells per call; a one-cell host-memory collide at N = 16 takes
 * 99 us under it against 447 us under the throughput schedule.  With auto the
 * summation order depends on the batch size, so results are reproducible per
 * batch size only.
 * Under the throughput schedule collide / RK2 at N >= 8 use the Hermitian
 * mirror schedule (conv.cuh k_conv_mirror2, with TMEM accumulators, at
 * N = 8, 12, 16; the phased k_conv_kcsm + k_conv_kcsr at N = 24, 32; env
 * BOLTZ_MIRROR=0 disables it, BOLTZ_MIRROR=1 selects k_conv_mirror, the
 * register-only variant, at N <= 16).
 * Results are bitwise reproducible and independent of batch composition
 * within a schedule; schedules differ by round-off.
 */
int boltz_set_schedule(boltz_ctx* ctx, int schedule);
/*
 * Executed K2 terms per cell eval: *plain for the throughput / latency
 * schedules and evaluate_qhat, *mirror for collide / RK2 when the Hermitian
 * mirror schedule is active (0 if not: N < 8, or a table that is not
 * mirror-symmetric).
 * Each is the size of its folded table, i.e. every FP64 term the kernel runs.
 */
int boltz_schedule_terms(boltz_ctx* ctx, int64_t* plain, int64_t* mirror);
/* Name of the K2 kernel(s) collide / RK2 run under the current schedule (for
 * the benchmark's roofline label; "" for a null context). */
const char* boltz_conv_kernel(const boltz_ctx* ctx);
int boltz_set_async(boltz_ctx* ctx, int enable);
int boltz_sync(boltz_ctx* ctx, void* stream);

/* ---- measurement hooks (bench.py; no reference counterpart) ---- */

/* Enable CUDA-event bracketing of every kernel launch on its stream.  Kinds:
 * 0 convolution (K2), 1 FFT passes (K1/K3), 2 projection/RK2 epilogue (K3),
 * 3 layout conversion, 4 transport (K4).  Launch counts are always kept. */
int boltz_set_timing(boltz_ctx* ctx, int enable);
/* ms[k], launches[k] for k < nkinds (nullable); reset != 0 zeroes them */
int boltz_get_timing(boltz_ctx* ctx, double* ms, int64_t* launches, int nkinds, int reset);
/* FP64 (DFMA) throughput of `device` in TFLOP/s, best over ~`seconds` */
int boltz_fp64_peak(int device, double seconds, double* tflops);

/* ---- host-side weight table (the hot path's input) ---- */

/* generate the dense zeta-major table (n^6 doubles) on the host; lambda in
 * {0,1} closed form, else composite Gauss-Legendre with `panels` panels. */
int boltz_generate_table(int n, double L, double lambda, double beta, double r0, int panels, double* G,
                         int nthreads);
double boltz_weight(double lambda, double beta, double r0, const double xi[3], const double zeta[3], int panels);

/* cache file: header (magic, version, N, L, lambda, beta, r0, panels) + LE doubles */
int boltz_save_table(const char* path, int n, double L, double lambda, double beta, double r0, int panels,
                     const double* G);
/* expected parameters must match the header exactly; G must hold n^6 doubles */
int boltz_load_table(const char* path, int n, double L, double lambda, double beta, double r0, int panels,
                     double* G);

/* ---- halo exchange of the sharded spatial domain (SURVEY §8b
 * "halo_exchange(...)", §8e), NCCL over NVLink / NVSwitch ---- */
#define BOLTZ_HALO_ID_BYTES 128
typedef struct boltz_halo boltz_halo;

/* rank 0 makes the communicator id and shares it out of band (one process per GPU) */
int boltz_halo_unique_id(unsigned char id[BOLTZ_HALO_ID_BYTES]);
/* ncclCommInitRank on `device` (collective over the `world` ranks) */
int boltz_halo_create(int rank, int world, const unsigned char id[BOLTZ_HALO_ID_BYTES], int device,
                      boltz_halo** out);
/* one process driving `world` GPUs (ncclCommInitAll): out[r] for devices[r] */
int boltz_halo_create_all(int world, const int* devices, boltz_halo** out);
int boltz_halo_destroy(boltz_halo* halo);
/*
 * Replaces halo_exchange: field is the
 * rank's DEVICE (ncl + 4) x n3 array; sends cells 2,3 left and ncl, ncl+1
 * right, receives into ghosts 0,1 and ncl+2, ncl+3 -- one grouped NCCL call,
 * one contiguous 2*n3 message per direction, ordered on `stream`.  The end
 * ranks leave their physical-end ghosts to boltz_fill_boundary.  Collective:
 * every rank calls it.
 */
int boltz_halo_exchange(boltz_halo* halo, double* field, int64_t ncl, int64_t n3, void* stream);
/* in-place sum over ranks of `count` device doubles (the conservation ledger) */
int boltz_halo_allreduce_sum(boltz_halo* halo, double* buf, int64_t count, void* stream);
/* in-process loopback backend: fields[r] are device arrays of
 * (ncl[r] + 4) x n3 on one device; copies every rank pair's ghosts */
int boltz_halo_exchange_loopback(double* const* fields, const int64_t* ncl, int nranks, int64_t n3, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BOLTZ_CUDA_H */
