/*
 * paratime_b200 — C ABI of the B200 (sm_100a) hot path of data-driven theta-parareal
 * for u_tt = c^2(x) Lap u on periodic 1D/2D boxes (arXiv 1905.00473).
 *
 * The reference ("paratime", /root/reference/proj) has no FFI; its boundary is the C++
 * header API in proj/include/paratime/*.hpp.  This header is the thin extern "C" layer
 * the C++ drop-in (include/paratime/*.hpp, same namespace and signatures) and any
 * foreign binding (ctypes) call.  Plain pointers and sizes only.
 *
 * Conventions (mirroring proj/include/paratime/grid.hpp:8-13):
 *   - fields are flat row-major fp64 arrays, 2D axis 0 = y (slow), axis 1 = x (fast);
 *   - a batch of B states is slice-major SoA: u[b*N + i], udot[b*N + i], N = grid size;
 *   - "_dev" pointers are device (HBM) addresses on the context's device, "_host"
 *     pointers are host memory (pinned or pageable);
 *   - every call is stream-ordered on the context stream.  Calls whose outputs are all
 *     device memory return without waiting for the GPU (like a CUDA library call: compose
 *     them freely, ptb_context_synchronize before reading results on the host); calls with
 *     host outputs (*_host, keep counts, residuals, ranks) complete before they return.
 * Errors: a ptb_status is returned and a thread-local message is kept
 * (ptb_last_error).  The C++ layer rethrows the reference's exception types:
 *   PTB_INVALID_ARGUMENT -> std::invalid_argument, PTB_DIVERGED -> PropagationDiverged,
 *   PTB_DOMAIN -> std::domain_error, others -> std::runtime_error.
 */
#ifndef PARATIME_B200_H_
#define PARATIME_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PTB_OK = 0,
  PTB_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  PTB_DIVERGED = 2,         /* PropagationDiverged (errors.hpp:9-12)   */
  PTB_DOMAIN = 3,           /* std::domain_error (energy_map.cpp:233)   */
  PTB_CUDA = 4,             /* CUDA runtime / cuBLAS failure            */
  PTB_NCCL = 5,             /* collective failure                       */
  PTB_UNSUPPORTED = 6,
  PTB_CONFIG = 7            /* ConfigError (errors.hpp): malformed input file */
} ptb_status;

/* Grid (grid.hpp:16-38): dim 1 or 2; n[0]/h[0] = axis 0 (y in 2D, the only axis in 1D). */
typedef struct {
  int dim;
  size_t n[2];
  double h[2];
} ptb_grid;

/* Propagator arithmetic.  EXACT reproduces propagator.cpp:31-73 operation by operation
 * (no FMA contraction) and is bitwise equal to the reference; FAST is the same velocity
 * Verlet in kick-drift-kick form with fused multiply-adds (parity <= 1e-12 rel. L2). */
typedef enum { PTB_MODE_FAST = 0, PTB_MODE_EXACT = 1 } ptb_mode;

typedef enum { PTB_INTERP_FOURIER = 0, PTB_INTERP_LINEAR = 1 } ptb_interp;     /* grid.hpp:54 */
typedef enum { PTB_FD2 = 0, PTB_FD4 = 1, PTB_FD6 = 2, PTB_FD8 = 3, PTB_SPECTRAL = 4 } ptb_scheme; /* energy_map.hpp:12 */

typedef struct ptb_context ptb_context;
typedef struct ptb_comm ptb_comm;
typedef struct ptb_propagator ptb_propagator;
typedef struct ptb_transfer ptb_transfer;

const char* ptb_last_error(void);
const char* ptb_version(void);

/* ---- context: device, stream, workspace --------------------------------------- */
ptb_status ptb_context_create(int device, ptb_context** out);
ptb_status ptb_context_destroy(ptb_context* ctx);
ptb_status ptb_context_synchronize(ptb_context* ctx);
/* cudaStream_t of the context (as void*); kernels of this context run on it */
void* ptb_context_stream(ptb_context* ctx);
/* run this context's work on an external cudaStream_t (e.g. the caller's current
 * stream; 0 = the legacy default stream) ... */
ptb_status ptb_context_set_stream(ptb_context* ctx, void* stream);
/* ... or back on the context's own non-blocking stream */
ptb_status ptb_context_use_own_stream(ptb_context* ctx);
int ptb_context_device(ptb_context* ctx);
/* number of this library's kernels launched on the context so far */
uint64_t ptb_context_launches(ptb_context* ctx);
ptb_status ptb_device_alloc(ptb_context* ctx, size_t bytes, void** out);
ptb_status ptb_device_free(ptb_context* ctx, void* p);
ptb_status ptb_memcpy_h2d(ptb_context* ctx, void* dst_dev, const void* src_host, size_t bytes);
ptb_status ptb_memcpy_d2h(ptb_context* ctx, void* dst_host, const void* src_dev, size_t bytes);

/* ---- propagator (propagator.hpp:12-31) ----------------------------------------- */
/* PropagatorConfig: validates exactly as propagator.cpp:11-27 (CFL, dt, steps) and
 * uploads the speed field c (host, N values) plus derived coefficient arrays. */
ptb_status ptb_propagator_create(ptb_context* ctx, const ptb_grid* grid, const double* c_host,
                                 double dt, size_t steps_per_coupling, ptb_propagator** out);
ptb_status ptb_propagator_destroy(ptb_propagator* p);
/* device speed array (N doubles) owned by the propagator */
const double* ptb_propagator_speed(ptb_propagator* p);

/* K1: steps_per_coupling Verlet steps on `batch` states in place (device pointers).
 * nonfinite_dev (nullable, int32[batch]) receives 1 where the result is not finite —
 * the condition on which propagate_coupling throws (propagator.cpp:102-103). */
ptb_status ptb_propagate_batch(ptb_propagator* p, size_t batch, double* u_dev, double* udot_dev,
                               int32_t* nonfinite_dev, int mode);
/* same with an explicit step count (used for `step`, propagator.cpp:85-93) */
/* Describe the launch plan propagate would use for (steps, batch, mode): kernel names, strip
 * widths and grids, NUL-terminated into buf (truncated to len).  Diagnostics only (new). */
ptb_status ptb_propagate_plan(ptb_propagator* p, size_t steps, size_t batch, int mode, char* buf, size_t len);

ptb_status ptb_propagate_steps_batch(ptb_propagator* p, size_t steps, size_t batch, double* u_dev,
                                     double* udot_dev, int32_t* nonfinite_dev, int mode);
/* propagate_coupling on host buffers (one state); PTB_DIVERGED when not finite. */
ptb_status ptb_propagate_coupling_host(ptb_propagator* p, const double* u_in, const double* udot_in,
                                       double* u_out, double* udot_out, int mode);
/* batched propagate_coupling on HOST buffers: H2D copy, K1, D2H copy, all stream-ordered
 * and chunked so copies of one chunk overlap the kernel of another.  nonfinite_host
 * (nullable, int32[batch]) gets the per-slice divergence flags. */
ptb_status ptb_propagate_batch_host(ptb_propagator* p, size_t batch, const double* u_in, const double* udot_in,
                                    double* u_out, double* udot_out, int32_t* nonfinite_host, int mode);
/* ---- absorbing layer (PML) fine propagator: BASELINE.json config 4 (not in the reference) --
 * The reference propagator is periodic only (propagator.cpp:31-105); SURVEY.md 8(f) rank 4.
 * State per slice: u, udot and the auxiliary fields px, py (same SoA layout); px, py must be
 * zero wherever zeta_x = zeta_y = 0.  Scheme: oracle/pml_np.py.  A zero profile reproduces the
 * periodic FAST propagator bitwise. */
typedef struct ptb_pml ptb_pml;
/* quadratic damping profile of `width` cells at both ends of an axis of n cells (host) */
ptb_status ptb_pml_damping_profile(size_t n, size_t width, double h, double cmax, double reflection,
                                   double* out_host);
/* validates like ptb_propagator_create (2D only); zeta_y_host: n[0] values, zeta_x_host: n[1] */
ptb_status ptb_pml_create(ptb_context* ctx, const ptb_grid* grid, const double* c_host,
                          const double* zeta_y_host, const double* zeta_x_host, double dt,
                          size_t steps_per_coupling, ptb_pml** out);
ptb_status ptb_pml_destroy(ptb_pml* p);
/* `steps` (0 = steps_per_coupling) steps on `batch` states in place (device pointers);
 * nonfinite_dev (nullable, int32[batch]) |= 1 where the result is not finite */
ptb_status ptb_pml_propagate_batch(ptb_pml* p, size_t steps, size_t batch, double* u_dev, double* udot_dev,
                                   double* px_dev, double* py_dev, int32_t* nonfinite_dev);
/* Plain parareal (Eq. 2, parareal.cpp:201-237) with the absorbing layer: states carry
 * (u, udot, px, py); fine and coarse are PML propagators on t's fine / coarse grids (the same
 * coupling interval); iterate 0 is the interpolated serial coarse chain, the sweep runs on the
 * coarse grid (R(I(d)) = d).  Host outputs (all nullable): rel_err_host[K x (N+1)] L2 distance of
 * [u; udot] to the serial fine run relative to the initial state's norm (the layer drains energy), iteration_ms_host[K] device time of each iteration body
 * (metrics excluded), states_host[4 x (N+1) x N_f] the last iterate, diverged_host = any
 * non-finite fine stage.  The theta (Procrustes) coupling: ptb_pml_theta_run below. */
ptb_status ptb_pml_parareal_run(ptb_pml* fine, ptb_pml* coarse, ptb_transfer* t, size_t n_couplings, int iterations,
                                const double* u0_host, const double* udot0_host, double* rel_err_host,
                                double* iteration_ms_host, double* states_host, int32_t* diverged_host);
/* the same with slices block-sharded over the ranks of `comm` (one all-gather of the coarse payload
 * per iteration, the last own fine state to the next rank); every rank gets the full error table,
 * states_host is filled for the rank's own states only.  Bitwise independent of the world size. */
ptb_status ptb_pml_parareal_run_sharded(ptb_pml* fine, ptb_pml* coarse, ptb_transfer* t, ptb_comm* comm,
                                        size_t n_couplings, int iterations, const double* u0_host,
                                        const double* udot0_host, double* rel_err_host, double* iteration_ms_host,
                                        double* states_host, int32_t* diverged_host);
/* Theta parareal (the data-driven Procrustes coupling, parareal.cpp:255-350) with the absorbing
 * layer — this build's extension (the reference defines the coupling on the periodic (u, udot)
 * state only, energy_map.cpp:137-214; scheme: oracle/pml_np.py theta_parareal).  The corrector is
 * fitted on Lambda of the (u, udot) snapshots (coarse speed of `coarse`, gradient `scheme`,
 * truncation `tol`); the sweep corrects (u, udot) through Lambda-dagger Omega Lambda and the
 * auxiliary fields additively.  comm nullable (one GPU).  Outputs as ptb_pml_parareal_run plus
 * ranks_host[K] (corrector rank) and residual_host[K] (relative_residual of the fit), nullable. */
ptb_status ptb_pml_theta_run(ptb_pml* fine, ptb_pml* coarse, ptb_transfer* t, ptb_comm* comm, size_t n_couplings,
                             int iterations, double tol, int scheme, const double* u0_host, const double* udot0_host,
                             double* rel_err_host, double* iteration_ms_host, double* states_host,
                             int32_t* ranks_host, double* residual_host, int32_t* diverged_host);
/* laplacian (propagator.cpp:31-58, reference operation order) */
ptb_status ptb_laplacian_batch(ptb_context* ctx, const ptb_grid* grid, size_t batch,
                               const double* f_dev, double* out_dev);

/* ---- grid transfer (grid.hpp:56-89) ----------------------------------------------- */
ptb_status ptb_transfer_create(ptb_context* ctx, const ptb_grid* coarse, const ptb_grid* fine,
                               int kind, ptb_transfer** out);
ptb_status ptb_transfer_destroy(ptb_transfer* t);
/* restrict_field: out[j] = in[ratio*j]; `batch` fields, slice-major */
ptb_status ptb_restrict_batch(ptb_transfer* t, size_t batch, const double* fine_dev, double* coarse_dev);
/* interpolate_field (trigonometric with split Nyquist, or periodic linear) */
ptb_status ptb_interpolate_batch(ptb_transfer* t, size_t batch, const double* coarse_dev, double* fine_dev);
/* out = base + I(coarse) for `batch` fields (the parareal combine next = fine_next + I(d));
 * base and out may alias */
ptb_status ptb_interpolate_add_batch(ptb_transfer* t, size_t batch, const double* coarse_dev, const double* base_dev,
                                     double* out_dev);
/* finite check of `batch` fields of n values each; flags_dev[b] |= 1 when any is non-finite */
ptb_status ptb_nonfinite_batch(ptb_context* ctx, size_t n, size_t batch, const double* f_dev,
                               int32_t* flags_dev);

/* ---- energy map (energy_map.hpp:32-53) ----------------------------------------------- */
/* Lambda: `batch` states -> stacked columns [grad axis 0; (grad axis 1;) udot/c] (column b at
 * stacked_dev + b*ld) and mean_u[b] = sum(u) (nullable).  c_dev: speed on `grid`. */
ptb_status ptb_energy_components_batch(ptb_context* ctx, const ptb_grid* grid, const double* c_dev, int scheme,
                                       size_t batch, const double* u_dev, const double* udot_dev,
                                       double* stacked_dev, size_t ld, double* mean_dev);
/* Lambda-dagger (from_energy_components): stacked columns + mean_u -> states */
ptb_status ptb_from_energy_components_batch(ptb_context* ctx, const ptb_grid* grid, const double* c_dev,
                                            size_t batch, const double* stacked_dev, size_t ld,
                                            const double* mean_dev, double* u_dev, double* udot_dev);
/* per state pair b: sums4[4b..] = {|Lambda(a-b)|^2, |Lambda(b)|^2, |u_a-u_b|^2, |u_b|^2}; energy,
 * energy_error and l2_error (energy_map.cpp:216-249) are closed forms of these sums */
ptb_status ptb_energy_sums_batch(ptb_context* ctx, const ptb_grid* grid, const double* c_dev, int scheme,
                                 size_t batch, const double* ua_dev, const double* udota_dev, const double* ub_dev,
                                 const double* udotb_dev, double* sums4_dev);
/* in-place complex DFT of `batch` fields (interleaved re/im), fft.hpp conventions */
ptb_status ptb_dft_batch(ptb_context* ctx, const ptb_grid* grid, size_t batch, double* data_dev, int inverse);

/* ---- Procrustes corrector (procrustes.hpp:22-81) ----------------------------------------- */
typedef struct ptb_corrector ptb_corrector;
/* an empty corrector (no accumulated data yet) */
ptb_status ptb_corrector_create(ptb_context* ctx, ptb_corrector** out);
ptb_status ptb_corrector_destroy(ptb_corrector* c);
/* update_svd (procrustes.cpp:188-237) in place; F, G: rows x cols column-major device, ld = rows */
ptb_status ptb_corrector_update(ptb_corrector* c, size_t rows, size_t cols, const double* F_dev, const double* G_dev,
                                double tol);
/* procrustes_solve (procrustes.cpp:177-186): validates shapes, then solves into c (reset) */
ptb_status ptb_procrustes_solve(ptb_corrector* c, size_t rows, size_t cols, const double* F_dev, const double* G_dev,
                                double tol);
ptb_status ptb_corrector_shape(ptb_corrector* c, size_t* rows, size_t* rank);
/* load factors from host (X, Y rows x rank column-major, S rank) — the value-type C++ API
 * keeps PhaseCorrector on the host and uploads it for each device operation */
ptb_status ptb_corrector_set(ptb_corrector* c, size_t rows, size_t rank, const double* X_host, const double* S_host,
                             const double* Y_host, double tol);
/* copy factors to host: X, Y rows x rank column-major, S rank */
ptb_status ptb_corrector_factors(ptb_corrector* c, double* X_host, double* S_host, double* Y_host);
/* out = copy with the first `count` triplets dropped (drop_leading) */
ptb_status ptb_corrector_drop_leading(ptb_corrector* c, size_t count, ptb_corrector** out);
/* out[:, b] = X (Y^T in[:, b]) for `batch` columns of length rows (apply, procrustes.cpp:82-86) */
ptb_status ptb_corrector_apply_batch(ptb_corrector* c, size_t batch, const double* in_dev, double* out_dev);
ptb_status ptb_relative_residual(ptb_corrector* c, size_t rows, size_t cols, const double* F_dev,
                                 const double* G_dev, double* out);

/* C (m x n) = alpha op(A) op(B) + beta C, column-major device arrays (BLAS dgemm semantics,
 * ta/tb: 1 = transposed).  The hand-written sm_100a DGEMM/DGEMV every corrector product uses
 * (procrustes.cpp:65-66, 201-234, 251; apply :82-86), exposed for parity tests and benchmarks. */
ptb_status ptb_dgemm(ptb_context* ctx, int ta, int tb, int m, int n, int k, double alpha, const double* A_dev,
                     int lda, const double* B_dev, int ldb, double beta, double* C_dev, int ldc);

/* building blocks of update_svd, exposed for parity tests:
 * truncated_qr (procrustes.cpp:34-46): A m x n (device, col-major) -> Q m x keep, R keep x n
 * (un-pivoted), keep = leading pivoted |R_ii| > drop_tol.  Q_dev/R_dev sized m*n / n*n. */
ptb_status ptb_truncated_qr(ptb_context* ctx, size_t m, size_t n, const double* A_dev, double drop_tol,
                            double* Q_dev, double* R_dev, size_t* keep);
/* thin SVD M (p x q) = U diag(S) V^T, k = min(p, q), S descending (S_host k values) */
ptb_status ptb_thin_svd(ptb_context* ctx, size_t p, size_t q, const double* M_dev, double* U_dev, double* S_host,
                        double* V_dev);

/* ---- speed-model text format (experiment.hpp:84-90, experiment.cpp:711-784) — host only ---- */
/* Writes "ny nx dy dx" then ny rows of nx values (%.17g).  needed = bytes required incl. NUL;
 * writes nothing when len < needed. */
ptb_status ptb_speed_model_write(const ptb_grid* grid, const double* c, char* buf, size_t len, size_t* needed);
/* Parses text; grid and (when cap >= points) c are filled; npoints = ny*nx.  PTB_CONFIG on
 * malformed input (the reference's ConfigError, message in ptb_last_error()). */
ptb_status ptb_speed_model_read(const char* text, ptb_grid* grid, double* c, size_t cap, size_t* npoints);

/* run-record CSV schemas of the reference's harness (experiment.cpp:596-628, write_run_files):
 * which = 0 errors.csv, 1 residuals.csv (header only when plain), 2 summary.csv, for K = iterations
 * records x couplings values (row-major energy_err, l2_err; per record residual, rank, diverged).
 * Host only.  Replaces: the reference writes these files only from run_experiment (no API). */
ptb_status ptb_run_csv(size_t iterations, size_t couplings, const double* energy_err, const double* l2_err,
                       const double* residual, const int* rank, const int* diverged, int plain, int which, char* buf,
                       size_t len, size_t* needed);

/* ---- parareal drivers (parareal.hpp:60-79) -------------------------------------------- */
typedef enum { PTB_PLAIN = 0, PTB_THETA = 1, PTB_CORRECTED_COARSE_ONLY = 2, PTB_OMEGA_IDENTITY = 3 } ptb_variant;

/* A CouplingSchedule + GridTransfer + options (parareal.hpp:17-57, experiment.hpp:20-44). */
typedef struct {
  int dim;
  size_t fine_n[2];
  double fine_h[2];
  size_t coarse_n[2];
  double coarse_h[2];
  double dt_fine;
  size_t m_fine;
  double dt_coarse;
  size_t m_coarse;
  double T;
  double dt_com;
  size_t n_couplings;
  int interp;         /* ptb_interp */
  int iterations;     /* K correction passes */
  int variant;        /* ptb_variant */
  int scheme;         /* data-matrix gradient (ThetaOptions::scheme) */
  int metric_scheme;  /* error seminorm (DriverOptions::metric_scheme) */
  double tol;         /* truncation tolerance */
  int remove_leading; /* singular triplets dropped before each sweep */
  int mode;           /* ptb_mode of the fine and coarse propagators */
} ptb_run_spec;

#define PTB_MAX_TIMED_ITERS 64
/* device-timed phases per iteration k = 1..K (CUDA events on the context stream) */
typedef struct {
  double reference_ms; /* serial fine reference (once per run) */
  double gather_ms[PTB_MAX_TIMED_ITERS];  /* coarse payload all-gather (0 on one GPU) */
  double parallel_ms[PTB_MAX_TIMED_ITERS];
  double procrustes_ms[PTB_MAX_TIMED_ITERS];
  double sweep_ms[PTB_MAX_TIMED_ITERS];
  double finalize_ms[PTB_MAX_TIMED_ITERS];
  double iteration_ms[PTB_MAX_TIMED_ITERS];
} ptb_phase_times;

/* plain_parareal / theta_parareal / corrected_coarse_only on one device.  Host inputs:
 * c_fine (fine N), c_coarse (coarse N), init (u0, udot0 on the fine grid).  Outputs (host):
 * energy_err, l2_err: (K+1)*(N+1) row-major [k][n]; residual, rank, diverged: K+1;
 * states (nullable): (K+1)*(N+1)*2*Nf as [k][n][u|udot][pt]; reference (nullable): (N+1)*2*Nf;
 * times (nullable). */
ptb_status ptb_parareal_run(ptb_context* ctx, const ptb_run_spec* spec, const double* c_fine,
                            const double* c_coarse, const double* u0, const double* udot0, double* energy_err,
                            double* l2_err, double* residual, int* rank, int* diverged, double* states,
                            double* reference, ptb_phase_times* times);

/* ---- multi-GPU (one process per GPU, NCCL over NVLink/NVSwitch) ----------------------- */
/* 128-byte ncclUniqueId created on rank 0 and broadcast by the caller (e.g. torch.distributed) */
ptb_status ptb_nccl_unique_id(char* out128);
ptb_status ptb_comm_create(ptb_context* ctx, int rank, int world, const char* id128, ptb_comm** out);
ptb_status ptb_comm_destroy(ptb_comm* c);
/* in-process ranks (one host thread per rank, contexts on the same or peer GPUs): the
 * collectives rendezvous on the host and copy with cudaMemcpy — for tests and single-node
 * debugging of the sharded driver */
ptb_status ptb_loopback_group_create(int world, void** out);
ptb_status ptb_loopback_group_destroy(void* group);
ptb_status ptb_comm_create_loopback(ptb_context* ctx, void* group, int rank, ptb_comm** out);

/* ptb_parareal_run with the N slices block-sharded over the ranks of `comm` (null = one GPU).
 * Every rank passes the same inputs; outputs energy_err/l2_err/residual/rank/diverged are
 * complete on every rank; states (nullable) receive this rank's slices only (plus n = 0
 * on rank 0).  Per iteration: one all-gather of the coarse per-slice payload, one of the
 * error sums, one boundary fine state to the next rank. */
ptb_status ptb_parareal_run_sharded(ptb_context* ctx, ptb_comm* comm, const ptb_run_spec* spec,
                                    const double* c_fine, const double* c_coarse, const double* u0,
                                    const double* udot0, double* energy_err, double* l2_err, double* residual,
                                    int* rank, int* diverged, double* states, double* reference,
                                    ptb_phase_times* times);

/* ---- measurement helpers (bench.py) ---------------------------------------------- */
/* Peak fp64 FMA throughput of the device: independent DFMA chains on every SM, timed
 * with CUDA events; returns TFLOP/s (2 flops per FMA) and the kernel time. */
ptb_status ptb_probe_fp64_peak(ptb_context* ctx, double* tflops, double* ms);

#ifdef __cplusplus
}
#endif

#endif /* PARATIME_B200_H_ */
