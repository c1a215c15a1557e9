// extern "C" entry points for the energy map, the Procrustes corrector and the drivers.
#include <cuda_runtime.h>

#include <algorithm>
#include <memory>

#include "ptb_comm.h"
#include "ptb_driver.h"
#include "ptb_energy.h"
#include "ptb_fft.h"
#include "ptb_procrustes.h"

struct ptb_corrector {
  ptb_context* ctx;
  ptb::DevCorrector c;
  std::unique_ptr<ptb::ProcWork> work;
};

using namespace ptb;

namespace {
struct Dev {
  int prev = -1;
  explicit Dev(int d) {
    cudaGetDevice(&prev);
    if (prev != d) cudaSetDevice(d);
  }
  ~Dev() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
}  // namespace

extern "C" {

ptb_status ptb_energy_components_batch(ptb_context* ctx, const ptb_grid* grid, const double* c, int scheme,
                                       size_t batch, const double* u, const double* v, double* stacked, size_t ld,
                                       double* mean) {
  return guarded([&] {
    require(ctx && grid, "energy_components: null argument");
    validate_grid(*grid);
    require(scheme >= PTB_FD2 && scheme <= PTB_SPECTRAL, "unknown gradient scheme");
    Dev d(ctx->device);
    std::lock_guard<std::recursive_mutex> lock(ctx->mutex);
    EnergyWork& w = context_energy_work(ctx);  // cached: no allocation (and no implicit sync) per call
    energy_components(w, *grid, scheme, batch, u, v, grid_size(*grid), nullptr, c, stacked, ld, mean);
  });
}

ptb_status ptb_from_energy_components_batch(ptb_context* ctx, const ptb_grid* grid, const double* c, size_t batch,
                                            const double* stacked, size_t ld, const double* mean, double* u,
                                            double* v) {
  return guarded([&] {
    require(ctx && grid, "from_energy_components: null argument");
    validate_grid(*grid);
    Dev d(ctx->device);
    std::lock_guard<std::recursive_mutex> lock(ctx->mutex);
    EnergyWork& w = context_energy_work(ctx);  // cached: no allocation (and no implicit sync) per call
    from_energy_components(w, *grid, batch, stacked, ld, mean, c, u, v, grid_size(*grid));
  });
}

ptb_status ptb_energy_sums_batch(ptb_context* ctx, const ptb_grid* grid, const double* c, int scheme, size_t batch,
                                 const double* ua, const double* va, const double* ub, const double* vb,
                                 double* sums4) {
  return guarded([&] {
    require(ctx && grid, "energy_sums: null argument");
    validate_grid(*grid);
    Dev d(ctx->device);
    std::lock_guard<std::recursive_mutex> lock(ctx->mutex);
    EnergyWork& w = context_energy_work(ctx);  // cached: no allocation (and no implicit sync) per call
    const size_t n = grid_size(*grid);
    pair_energy_sums(w, *grid, scheme, batch, ua, va, n, ub, vb, n, c, sums4);
  });
}

ptb_status ptb_dft_batch(ptb_context* ctx, const ptb_grid* grid, size_t batch, double* data, int inverse) {
  return guarded([&] {
    require(ctx && grid, "dft: null argument");
    validate_grid(*grid);
    Dev d(ctx->device);
    fft_field(ctx, ctx->stream, *grid, batch, reinterpret_cast<double2*>(data), inverse != 0);
  });
}

ptb_status ptb_corrector_create(ptb_context* ctx, ptb_corrector** out) {
  return guarded([&] {
    require(ctx && out, "corrector: null argument");
    auto* c = new ptb_corrector();
    c->ctx = ctx;
    c->work = std::make_unique<ProcWork>(ctx);
    *out = c;
  });
}

ptb_status ptb_corrector_destroy(ptb_corrector* c) {
  return guarded([&] {
    if (!c) return;
    Dev d(c->ctx->device);
    delete c;
  });
}

ptb_status ptb_corrector_update(ptb_corrector* c, size_t rows, size_t cols, const double* F, const double* G,
                                double tol) {
  return guarded([&] {
    require(c != nullptr, "update_svd: null corrector");
    check_tol(tol);
    Dev d(c->ctx->device);
    std::lock_guard<std::recursive_mutex> lock(c->ctx->mutex);
    update_svd(*c->work, c->c, F, G, int(rows), int(cols), tol);
  });
}

ptb_status ptb_procrustes_solve(ptb_corrector* c, size_t rows, size_t cols, const double* F, const double* G,
                                double tol) {
  return guarded([&] {
    require(c != nullptr, "procrustes_solve: null corrector");
    check_tol(tol);
    require(cols <= rows, "procrustes_solve: more snapshots than rows");
    require(cols > 0, "procrustes_solve: empty data");
    Dev d(c->ctx->device);
    std::lock_guard<std::recursive_mutex> lock(c->ctx->mutex);
    solve_from_scratch(*c->work, c->c, F, G, int(rows), int(cols), tol);
  });
}

ptb_status ptb_corrector_set(ptb_corrector* c, size_t rows, size_t rank, const double* X, const double* S,
                             const double* Y, double tol) {
  return guarded([&] {
    require(c != nullptr, "corrector: null");
    require(rank == 0 || (X && S && Y), "corrector: null factors");
    Dev d(c->ctx->device);
    const size_t n = rows * rank;
    double* dx = static_cast<double*>(c->c.X.get(std::max<size_t>(1, n) * sizeof(double)));
    double* dy = static_cast<double*>(c->c.Y.get(std::max<size_t>(1, n) * sizeof(double)));
    if (n) {
      PTB_CUDA_CHECK(cudaMemcpy(dx, X, n * sizeof(double), cudaMemcpyHostToDevice));
      PTB_CUDA_CHECK(cudaMemcpy(dy, Y, n * sizeof(double), cudaMemcpyHostToDevice));
    }
    c->c.assign(int(rows), int(rank), std::vector<double>(S, S + rank), tol);
  });
}

ptb_status ptb_corrector_shape(ptb_corrector* c, size_t* rows, size_t* rank) {
  return guarded([&] {
    require(c && rows && rank, "corrector: null argument");
    *rows = size_t(c->c.rows);
    *rank = size_t(c->c.rank);
  });
}

ptb_status ptb_corrector_factors(ptb_corrector* c, double* X, double* S, double* Y) {
  return guarded([&] {
    require(c != nullptr, "corrector: null");
    Dev d(c->ctx->device);
    const size_t n = size_t(c->c.rows) * c->c.rank;
    if (n) {
      PTB_CUDA_CHECK(cudaMemcpy(X, c->c.Xp(), n * sizeof(double), cudaMemcpyDeviceToHost));
      PTB_CUDA_CHECK(cudaMemcpy(Y, c->c.Yp(), n * sizeof(double), cudaMemcpyDeviceToHost));
    }
    for (size_t i = 0; i < c->c.S.size(); ++i) S[i] = c->c.S[i];
  });
}

ptb_status ptb_corrector_drop_leading(ptb_corrector* c, size_t count, ptb_corrector** out) {
  return guarded([&] {
    require(c && out, "drop_leading: null argument");
    Dev d(c->ctx->device);
    auto* o = new ptb_corrector();
    o->ctx = c->ctx;
    o->work = std::make_unique<ProcWork>(c->ctx);
    drop_leading(c->c, count, o->c, c->ctx);
    *out = o;
  });
}

ptb_status ptb_corrector_apply_batch(ptb_corrector* c, size_t batch, const double* in, double* out) {
  return guarded([&] {
    require(c != nullptr, "apply: null corrector");
    Dev d(c->ctx->device);
    std::lock_guard<std::recursive_mutex> lock(c->ctx->mutex);
    apply_corrector(*c->work, c->c, batch, in, size_t(c->c.rows), out, size_t(c->c.rows));
  });
}

ptb_status ptb_dgemm(ptb_context* ctx, int ta, int tb, int m, int n, int k, double alpha, const double* A, int lda,
                     const double* B, int ldb, double beta, double* C, int ldc) {
  return guarded([&] {
    require(ctx && (m == 0 || n == 0 || (C && (k == 0 || (A && B)))), "dgemm: null argument");
    require(m >= 0 && n >= 0 && k >= 0 && ldc >= std::max(1, m), "dgemm: bad dimensions");
    require(lda >= std::max(1, ta ? k : m) && ldb >= std::max(1, tb ? n : k), "dgemm: leading dimension too small");
    Dev d(ctx->device);
    std::lock_guard<std::recursive_mutex> lock(ctx->mutex);
    gemm(ctx, ta != 0, tb != 0, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
  });
}

ptb_status ptb_relative_residual(ptb_corrector* c, size_t rows, size_t cols, const double* F, const double* G,
                                 double* out) {
  return guarded([&] {
    require(c && out, "relative_residual: null argument");
    Dev d(c->ctx->device);
    std::lock_guard<std::recursive_mutex> lock(c->ctx->mutex);
    *out = relative_residual(*c->work, c->c, F, G, int(rows), int(cols));
  });
}

ptb_status ptb_truncated_qr(ptb_context* ctx, size_t m, size_t n, const double* A, double drop_tol, double* Q,
                            double* R, size_t* keep) {
  return guarded([&] {
    require(ctx && keep, "truncated_qr: null argument");
    Dev d(ctx->device);
    std::lock_guard<std::recursive_mutex> lock(ctx->mutex);
    ProcWork& w = context_proc_work(ctx);
    DeviceBuffer& qb = w.QF;  // the workspace's own buffers: no allocation per call
    DeviceBuffer& rb = w.RF;
    const int k = truncated_qr(w, A, int(m), int(n), drop_tol, qb, rb);
    if (k > 0) {
      PTB_CUDA_CHECK(cudaMemcpyAsync(Q, qb.ptr, m * size_t(k) * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
      PTB_CUDA_CHECK(cudaMemcpyAsync(R, rb.ptr, size_t(k) * n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    }
    PTB_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    *keep = size_t(k);
  });
}

ptb_status ptb_thin_svd(ptb_context* ctx, size_t p, size_t q, const double* M, double* U, double* S, double* V) {
  return guarded([&] {
    require(ctx && S, "thin_svd: null argument");
    Dev d(ctx->device);
    std::lock_guard<std::recursive_mutex> lock(ctx->mutex);
    ProcWork& w = context_proc_work(ctx);
    DeviceBuffer& ub = w.Uh;
    DeviceBuffer& vb = w.Vh;
    std::vector<double> sigma;
    thin_svd(w, M, int(p), int(q), ub, sigma, vb);
    const size_t k = std::min(p, q);
    if (k) {
      PTB_CUDA_CHECK(cudaMemcpy(U, ub.ptr, p * k * sizeof(double), cudaMemcpyDeviceToDevice));
      PTB_CUDA_CHECK(cudaMemcpy(V, vb.ptr, q * k * sizeof(double), cudaMemcpyDeviceToDevice));
    }
    for (size_t i = 0; i < k; ++i) S[i] = sigma[i];
  });
}

ptb_status ptb_parareal_run(ptb_context* ctx, const ptb_run_spec* spec, const double* cf, const double* cc,
                            const double* u0, const double* v0, double* ee, double* l2, double* residual, int* rank,
                            int* diverged, double* states, double* reference, ptb_phase_times* times) {
  return guarded([&] {
    require(ctx && spec && cf && cc && u0 && v0 && ee && l2 && residual && rank && diverged,
            "parareal: null argument");
    Dev d(ctx->device);
    run_parareal(ctx, nullptr, *spec, cf, cc, u0, v0, ee, l2, residual, rank, diverged, states, reference, times);
  });
}

ptb_status ptb_parareal_run_sharded(ptb_context* ctx, ptb_comm* comm, const ptb_run_spec* spec, const double* cf,
                                    const double* cc, const double* u0, const double* v0, double* ee, double* l2,
                                    double* residual, int* rank, int* diverged, double* states, double* reference,
                                    ptb_phase_times* times) {
  return guarded([&] {
    require(ctx && spec && cf && cc && u0 && v0 && ee && l2 && residual && rank && diverged,
            "parareal: null argument");
    Dev d(ctx->device);
    run_parareal(ctx, comm_of(comm), *spec, cf, cc, u0, v0, ee, l2, residual, rank, diverged, states, reference,
                 times);
  });
}

}  // extern "C"
