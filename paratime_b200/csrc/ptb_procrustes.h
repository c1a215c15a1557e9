#pragma once
#include <functional>
#include <vector>

#include "ptb_internal.h"

namespace ptb {

// Device-resident truncated factors (X, S, Y) of the accumulated correlation matrix
// (procrustes.hpp:22-60): X, Y are rows x rank column-major in HBM, S on host + device.
struct DevCorrector {
  int rows = 0, rank = 0;
  double tol = 0.0;
  std::vector<double> S;
  DeviceBuffer X, Y, Sd;
  bool empty() const { return rows == 0; }
  const double* Xp() const { return static_cast<const double*>(X.ptr); }
  const double* Yp() const { return static_cast<const double*>(Y.ptr); }
  double* Xp() { return static_cast<double*>(X.ptr); }
  double* Yp() { return static_cast<double*>(Y.ptr); }
  void assign(int rows_, int rank_, const std::vector<double>& s, double tol_);
  DevCorrector() = default;
  DevCorrector(const DevCorrector&) = delete;
  DevCorrector& operator=(const DevCorrector&) = delete;
  ~DevCorrector();
};

struct ProcWork {
  ptb_context* ctx;
  DeviceBuffer buf[24];
  DeviceBuffer QF, RF, QG, RG, Uh, Vh;
  DeviceBuffer PQ, PR, PU;  // thin_svd preconditioning: Q, R of the QR and U of R^T
  DeviceBuffer SX, SY;      // spare corrector factors: update_svd writes here, then swaps
  DeviceBuffer BA, BV, BT, BR, BQ2;  // blocked tall QR: work copy, reflectors, tau/T/W, R1, Q2
  DeviceBuffer TS[24], TX[2];       // TSQR: per level reflectors, tau, R stack; Q down-sweep ping-pong
  DeviceBuffer TS2[24], TX2[2], BQ2b;  // the second matrix of a batched (F, G) TSQR
  DeviceBuffer PA[4], PB[4];        // batched TSQR: the two final pivoted factors, tau, perm, |R_jj|
  DeviceBuffer TP[8];               // two-panel TSQR: Q1, R1, A2, C, Q2, R2, the assembled R
  DeviceBuffer TPg[8];              // the second matrix (G) of the row-sharded two-panel pair
  DeviceBuffer SH[12];              // row-sharded update_svd: level-0 leaves, stacks, slab partials, gathers
  DeviceBuffer SG[6];               // the second matrix (G) of the row-sharded pair TSQR
  // the ranks the corrector's rows are sharded over (update_svd; null: one process).  Set by the
  // parareal driver around its update_svd call.
  const struct Comm* comm = nullptr;
  explicit ProcWork(ptb_context* c);
  ~ProcWork();
};

void check_tol(double tol);
int truncated_qr(ProcWork& w, const double* A, int m, int n, double drop_tol, DeviceBuffer& Q, DeviceBuffer& R);
void thin_svd(ProcWork& w, const double* M, int p, int q, DeviceBuffer& U, std::vector<double>& sigma, DeviceBuffer& V);
void solve_from_scratch(ProcWork& w, DevCorrector& out, const double* F, const double* G, int rows, int cols,
                        double tol);
void update_svd(ProcWork& w, DevCorrector& c, const double* F, const double* G, int rows, int cols, double tol);
void apply_corrector(ProcWork& w, const DevCorrector& c, size_t batch, const double* in, size_t ld_in, double* out,
                     size_t ld_out);
double relative_residual(ProcWork& w, const DevCorrector& c, const double* F, const double* G, int rows, int cols);
void drop_leading(const DevCorrector& c, size_t count, DevCorrector& out, ptb_context* ctx);
void gemm(ptb_context* ctx, bool ta, bool tb, int m, int n, int k, double alpha, const double* A, int lda,
          const double* B, int ldb, double beta, double* C, int ldc);
void geam_sub(ptb_context* ctx, size_t total, const double* F, double* D);  // D = F - D
// row-sharded corrector products (gemm.cu): row-local C = alpha A B + beta C (never split over k),
// and A^T B over fixed row slabs with the partials of slabs [z0, z0 + nz) computed here
void gemm_rows(ptb_context* ctx, int m, int n, int k, double alpha, const double* A, int lda, const double* B, int ldb,
               double beta, double* C, int ldc);
void gemm_tn_slabs(ptb_context* ctx, int m, int n, const double* A, int lda, const double* B, int ldb, double* C,
                   int ldc, int P, int slab, int z0, int nz, double* ws_own, double* ws_all,
                   const std::function<void()>& gather);
void fix_signs(ptb_context* ctx, double* X, double* Y, int rows, int cols);

}  // namespace ptb
