// Energy-norm Procrustes corrector on the device (K5/K6).
//
// Reference: /root/reference/proj/src/procrustes.cpp
//   check_tol            :14-17    tol in (0, 1)
//   fix_signs            :21-30    largest-|.| entry of each left column positive (first max)
//   truncated_qr         :34-46    column-pivoted thin QR, R un-pivoted, keep leading |R_ii| > guard
//   solve_from_scratch   :48-69    SVD(R_F R_G^T), keep sigma_i/sigma_1 > tol, X = Q_F U, Y = Q_G V
//   apply / drop_leading :82-93
//   update_svd           :188-237  Algorithm 1
//   relative_residual    :245-253
//
// Kernels written here (sm_100a):
//   truncated_qr   tall blocks (m >= 8n, n > 32): blocked Householder QR -- k_qr_panel (one
//                  panel of 32 columns, unpivoted, ONE grid barrier per column: the next
//                  column's norm and raw dot products are reduced during the current update)
//                  with compact-WY trailing updates (cuBLAS DGEMMs), then the column-pivoted
//                  QR of the small R1 (pivots and |R_jj| of A, since norms are invariant under
//                  Q1), Q = Q1 [Q2; 0].  Other shapes: k_qrcp (cooperative, rows split over
//                  CTAs, dgeqp3 pivot rule with exact norms) or k_qrcp_small (whole matrix in
//                  one CTA's shared memory).  Both stop at the first |R_jj| <= guard.
//   k_wy_prep / k_wy_larft + DGEMMs   thin Q in compact WY form (dlarft / dorg2r order).
//   k_jacobi       one-sided (Hestenes) Jacobi SVD in a single CTA (shared memory when it fits),
//                  round-robin pairs, relative-orthogonality stop; k_jacobi_coop spreads the same
//                  schedule over a cooperative grid (bitwise equal) for larger matrices.  thin_svd
//                  preconditions with a pivoted QR (Jacobi on R^T, as dgesvj).
//   k_fix_signs    one CTA per column.
// Large products (U^T F, U UF, [U Q_F] Xh, X(Y^T v)) are plain cuBLAS DGEMMs.

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "ptb_dsmem.h"
#include "ptb_comm.h"
#include "ptb_procrustes.h"

namespace cg = cooperative_groups;

namespace ptb {
namespace {

constexpr int QR_THREADS = 1024;

struct QrArgs {
  double* A;  // m x n column-major, leading dimension lda (>= m)
  int m, n;
  int lda;
  int pivot;  // 0: no column pivoting (panels of the blocked QR)
  double drop_tol;
  double* tau;     // n
  int* perm;       // n (pivoted column j = original column perm[j])
  double* part;    // [2][grid][n+1] partial sums
  int* keep_out;   // 1
  double* beta_out;  // n (|R_jj| sequence, for diagnostics)
};

__device__ double cta_reduce(double x, double* red) {
  // fixed-order tree over QR_THREADS values
  red[threadIdx.x] = x;
  __syncthreads();
  for (int s = QR_THREADS / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

__device__ __forceinline__ double warp_sum(double x) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Values written by other CTAs (partial sums, the pivot row) are read with __ldcg: the
// grid barrier orders the writes but does not invalidate this SM's L1, so a plain load
// could return a line cached two steps earlier.  Per column step: one warp per trailing
// column computes its dot product / update over the CTA's rows and reduces with shuffles,
// so the only block-wide barriers are the three grid barriers.
__global__ void __launch_bounds__(QR_THREADS) k_qrcp(QrArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sh[];  // red[QR_THREADS] | w[n] | nrm[n] | vs[rows_per]
  double* red = sh;
  double* w = red + QR_THREADS;
  double* nrm = w + a.n;
  double* vs = nrm + a.n;  // this CTA's rows of the current reflector (1 at row j, 0 above)
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = QR_THREADS / 32;
  const int m = a.m, n = a.n;
  const int rows_per = (m + G - 1) / G;
  const int r0 = min(m, g * rows_per), r1 = min(m, r0 + rows_per);
  double* A = a.A;
  auto col = [&](int k) { return A + size_t(k) * a.lda; };
  for (int k = warp; k < n; k += nwarps) {  // initial squared column norms, per CTA
    double sacc = 0.0;
    for (int i = r0 + lane; i < r1; i += 32) sacc += col(k)[i] * col(k)[i];
    sacc = warp_sum(sacc);
    if (lane == 0) a.part[size_t(g) * (n + 1) + k] = sacc;
  }
  if (g == 0)
    for (int k = tid; k < n; k += QR_THREADS) a.perm[k] = k;
  int keep = 0;
  for (int j = 0; j < n && j < m; ++j) {
    double* part = a.part + size_t(j & 1) * G * (n + 1);
    double* partn = a.part + size_t((j + 1) & 1) * G * (n + 1);
    grid.sync();
    // cross-CTA partials: one warp per column, lanes over CTAs (fixed order for a given grid)
    for (int k = j + warp; k < n; k += nwarps) {
      double sacc = 0.0;
      for (int c = lane; c < G; c += 32) sacc += __ldcg(&part[size_t(c) * (n + 1) + k]);
      sacc = warp_sum(sacc);
      if (lane == 0) nrm[k] = sacc;
    }
    __syncthreads();
    int p = j;  // max remaining norm, first index on ties (idamax)
    if (a.pivot) {
      double best = nrm[j];
      for (int k = j + 1; k < n; ++k)
        if (nrm[k] > best) {
          best = nrm[k];
          p = k;
        }
    }
    if (p != j) {
      for (int i = r0 + tid; i < r1; i += QR_THREADS) {
        const double t = col(j)[i];
        col(j)[i] = col(p)[i];
        col(p)[i] = t;
      }
      if (g == 0 && tid == 0) {
        const int t = a.perm[j];
        a.perm[j] = a.perm[p];
        a.perm[p] = t;
      }
    }
    __syncthreads();
    // below-diagonal norm of the pivot column (dlarfg's xnorm) from its own partial
    double xs = 0.0;
    for (int i = max(r0, j + 1) + tid; i < r1; i += QR_THREADS) xs += col(j)[i] * col(j)[i];
    xs = cta_reduce(xs, red);
    if (tid == 0) partn[size_t(g) * (n + 1) + n] = xs;
    grid.sync();
    if (warp == 0) {
      double sacc = 0.0;
      for (int c = lane; c < G; c += 32) sacc += __ldcg(&partn[size_t(c) * (n + 1) + n]);
      sacc = warp_sum(sacc);
      if (lane == 0) red[0] = sacc;
    }
    __syncthreads();
    const double xnorm2 = red[0];
    __syncthreads();  // red is reused by cta_reduce in the next column
    const double alpha = __ldcg(&col(j)[j]);
    const double xnorm = sqrt(xnorm2);
    double beta, tau, scal;
    if (xnorm == 0.0) {
      beta = alpha;
      tau = 0.0;
      scal = 0.0;
    } else {
      beta = -copysign(hypot(alpha, xnorm), alpha);
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    if (fabs(beta) <= a.drop_tol) {  // first pivot at or below the guard: keep = j
      if (g == 0 && tid == 0) a.beta_out[j] = fabs(beta);
      break;
    }
    keep = j + 1;
    if (g == 0 && tid == 0) {
      a.tau[j] = tau;
      a.beta_out[j] = fabs(beta);
    }
    for (int i = r0 + tid; i < r1; i += QR_THREADS) {
      double x = 0.0;
      if (i > j) {
        x = col(j)[i] * scal;
        col(j)[i] = x;
      } else if (i == j) {
        x = 1.0;
      }
      vs[i - r0] = x;
    }
    __syncthreads();  // the dot products below read rows scaled by other threads
    const int i0 = max(r0, j);
    // w_k = v^T A[j:, k] over own rows; 4 independent accumulators keep 4 loads in flight per lane
    for (int k = j + 1 + warp; k < n; k += nwarps) {
      const double* ck = col(k);
      double s[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      int i = i0 + lane;
      for (; i + 224 < r1; i += 256) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = ck[i + 32 * u];
#pragma unroll
        for (int u = 0; u < 8; ++u) s[u] += vs[i + 32 * u - r0] * x[u];
      }
      for (; i < r1; i += 32) s[0] += vs[i - r0] * ck[i];
      const double sacc = warp_sum(((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7])));
      if (lane == 0) part[size_t(g) * (n + 1) + k] = sacc;
    }
    grid.sync();
    for (int k = j + 1 + warp; k < n; k += nwarps) {
      double sacc = 0.0;
      for (int c = lane; c < G; c += 32) sacc += __ldcg(&part[size_t(c) * (n + 1) + k]);
      sacc = warp_sum(sacc);
      if (lane == 0) w[k] = sacc;
    }
    __syncthreads();
    for (int k = j + 1 + warp; k < n; k += nwarps) {  // A[:, k] -= tau v w_k; fused next norms
      const double tw = tau * w[k];
      double* ck = col(k);
      double s[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      int i = i0 + lane;
      for (; i + 224 < r1; i += 256) {
        double x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = ck[i + 32 * u];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          x[u] -= tw * vs[i + 32 * u - r0];
          ck[i + 32 * u] = x[u];
        }
        s[0] += i != j ? x[0] * x[0] : 0.0;  // row j becomes R's row: not part of the trailing norms
#pragma unroll
        for (int u = 1; u < 8; ++u) s[u] += x[u] * x[u];
      }
      for (; i < r1; i += 32) {
        const double x = ck[i] - tw * vs[i - r0];
        ck[i] = x;
        if (i != j) s[0] += x * x;
      }
      const double sacc = warp_sum(((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7])));
      if (lane == 0) partn[size_t(g) * (n + 1) + k] = sacc;
    }
    __syncthreads();
    if (j >= r0 && j < r1 && tid == 0) col(j)[j] = beta;
  }
  if (g == 0 && tid == 0) *a.keep_out = keep;
}

// Column-pivoted Householder QR of a small matrix held entirely in one CTA's shared memory
// (the corrector's H and the blocked QR's R1: up to ~160 x 160).  Same algorithm, keep rule and
// output layout as k_qrcp (R above the diagonal with beta on it, scaled reflectors below, tau,
// perm, keep, |R_jj| sequence) without grid barriers or global-memory sweeps.
// SMEM = false: the same single-CTA kernel working in place on global memory (lda == m; the
// matrix stays L2-resident), for matrices too large for shared memory but small enough that one
// CTA without grid barriers beats the cooperative kernel (the corrector's H at cfg4, ~270^2).
template <bool SMEM>
__global__ void __launch_bounds__(1024) k_qrcp_small(QrArgs a) {
  extern __shared__ double qs[];  // SMEM: A[m*n] | nrm[n] | w[n] | red[32];  else nrm | w | red
  const int m = a.m, n = a.n, tid = threadIdx.x, T = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = T >> 5;
  double* A = SMEM ? qs : a.A;
  double* nrm = SMEM ? A + size_t(m) * n : qs;
  double* wv = nrm + n;
  double* red = wv + n;
  __shared__ int piv;
  __shared__ double s_xn2;
  if (SMEM)
    for (int e = tid; e < m * n; e += T) {
      const int c = e / m, i = e - c * m;
      A[e] = a.A[size_t(c) * a.lda + i];
    }
  for (int k = tid; k < n; k += T) a.perm[k] = k;
  __syncthreads();
  for (int k = warp; k < n; k += nwarps) {  // initial squared column norms
    double acc = 0.0;
    for (int i = lane; i < m; i += 32) acc += A[size_t(k) * m + i] * A[size_t(k) * m + i];
    acc = warp_sum(acc);
    if (lane == 0) nrm[k] = acc;
  }
  __syncthreads();
  int keep = 0;
  for (int j = 0; j < n && j < m; ++j) {
    if (warp == 0) {  // pivot: max remaining norm, first index on ties (idamax)
      double best = -1.0;
      int bi = n;
      for (int k = j + lane; k < n; k += 32)
        if (nrm[k] > best) {
          best = nrm[k];
          bi = k;
        }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      if (lane == 0) piv = bi;
    }
    __syncthreads();
    const int p = piv;
    if (p != j) {
      for (int i = tid; i < m; i += T) {
        const double t = A[size_t(j) * m + i];
        A[size_t(j) * m + i] = A[size_t(p) * m + i];
        A[size_t(p) * m + i] = t;
      }
      if (tid == 0) {
        const int t = a.perm[j];
        a.perm[j] = a.perm[p];
        a.perm[p] = t;
        const double tn = nrm[j];
        nrm[j] = nrm[p];
        nrm[p] = tn;
      }
      __syncthreads();
    }
    double* cj = A + size_t(j) * m;
    if (warp == 0) {  // below-diagonal norm of the pivot column (dlarfg's xnorm)
      double acc = 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) acc += cj[i] * cj[i];
      acc = warp_sum(acc);
      if (lane == 0) s_xn2 = acc;
    }
    __syncthreads();
    const double alpha = cj[j];
    const double xnorm = sqrt(s_xn2);
    double beta, tau, scal;
    if (xnorm == 0.0) {
      beta = alpha;
      tau = 0.0;
      scal = 0.0;
    } else {
      beta = -copysign(hypot(alpha, xnorm), alpha);
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    if (fabs(beta) <= a.drop_tol) {
      if (tid == 0) a.beta_out[j] = fabs(beta);
      break;
    }
    keep = j + 1;
    if (tid == 0) {
      a.tau[j] = tau;
      a.beta_out[j] = fabs(beta);
    }
    for (int i = j + 1 + tid; i < m; i += T) cj[i] *= scal;
    __syncthreads();
    for (int k = j + 1 + warp; k < n; k += nwarps) {  // w_k = v^T A[j:, k]
      const double* ck = A + size_t(k) * m;
      double acc = lane == 0 ? ck[j] : 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) acc += cj[i] * ck[i];
      acc = warp_sum(acc);
      if (lane == 0) wv[k] = acc;
    }
    __syncthreads();
    for (int k = j + 1 + warp; k < n; k += nwarps) {  // A[:, k] -= tau v w_k; next norms below row j
      double* ck = A + size_t(k) * m;
      const double tw = tau * wv[k];
      if (lane == 0) ck[j] -= tw;
      double acc = 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) {
        const double x = ck[i] - tw * cj[i];
        ck[i] = x;
        acc += x * x;
      }
      acc = warp_sum(acc);
      if (lane == 0) nrm[k] = acc;
    }
    if (tid == 0) cj[j] = beta;
    __syncthreads();
  }
  if (SMEM)
    for (int e = tid; e < m * n; e += T) {
      const int c = e / m, i = e - c * m;
      a.A[size_t(c) * a.lda + i] = A[e];
    }
  if (tid == 0) *a.keep_out = keep;
  (void)red;
}

// Unpivoted Householder QR of a tall panel (the blocked QR's panels) with ONE grid barrier per
// column: column j+1's squared norm and its raw dot products with the trailing columns are
// accumulated during column j's update pass (w_k = A_jk + scal * sum_{i>j} x_i A_ik needs only the
// unscaled column), so the reduction, the reflector and the update of a column need no further
// barrier.  Within a CTA, column j+1 is updated first, then (after a CTA barrier) every other
// trailing column is updated and dotted with it in the same sweep.  Partials are double-buffered
// by column parity.  Outputs as k_qrcp (LAPACK layout: R above, v below the diagonal, tau).
struct PanelArgs {
  double* A;
  int m, n, lda;
  double* tau;
  double* part;  // [2][grid][n + 1]: dots (k), squared norm (n)
  double* rowb;  // [2][n]: row j of the panel as of the start of column j (A_jj = alpha, A_jk)
};

__global__ void __launch_bounds__(QR_THREADS) k_qr_panel(PanelArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sh[];  // wv[n] | vs[rows_per] | xs[rows_per]
  const int G = gridDim.x, g = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, nwarps = QR_THREADS / 32;
  const int m = a.m, n = a.n;
  const int rows_per = (m + G - 1) / G;
  const int r0 = min(m, g * rows_per), r1 = min(m, r0 + rows_per);
  double* wv = sh;
  double* vs = wv + n;
  double* xs = vs + rows_per;
  auto col = [&](int k) { return a.A + size_t(k) * a.lda; };
  auto slot = [&](int j) { return a.part + size_t(j & 1) * G * (n + 1) + size_t(g) * (n + 1); };
  // row j is rewritten by its owner during column j's pass while other CTAs still need its
  // values, so the owner publishes a copy (parity j & 1) before the barrier that precedes use
  auto rowcopy = [&](int j) { return a.rowb + size_t(j & 1) * n; };
  if (r0 == 0 && r1 > 0)
    for (int k = tid; k < n; k += QR_THREADS) rowcopy(0)[k] = col(k)[0];
  // partials of column 0
  {
    double* P = slot(0);
    const double* x = col(0);
    for (int k = warp; k <= n; k += nwarps) {
      double acc = 0.0;
      if (k == n) {
        for (int i = max(r0, 1) + lane; i < r1; i += 32) acc += x[i] * x[i];
      } else if (k > 0) {
        const double* ck = col(k);
        for (int i = max(r0, 1) + lane; i < r1; i += 32) acc += x[i] * ck[i];
      }
      acc = warp_sum(acc);
      if (lane == 0) P[k] = acc;
    }
  }
  for (int j = 0; j < n && j < m; ++j) {
    grid.sync();
    const double* Pj = a.part + size_t(j & 1) * G * (n + 1);
    // reduce: squared norm below the diagonal (into wv[j]) and raw dots d_k (into wv[k], k > j)
    for (int k = j + warp; k <= n; k += nwarps) {
      if (k == j) continue;
      double acc = 0.0;
      for (int c = lane; c < G; c += 32) acc += __ldcg(&Pj[size_t(c) * (n + 1) + k]);
      acc = warp_sum(acc);
      if (lane == 0) wv[k == n ? j : k] = acc;
    }
    __syncthreads();
    const double xnorm2 = wv[j];
    const double* rowj = rowcopy(j);
    const double alpha = __ldcg(&rowj[j]);
    const double xnorm = sqrt(xnorm2);
    double beta, tau, scal;
    if (xnorm == 0.0) {
      beta = alpha;
      tau = 0.0;
      scal = 0.0;
    } else {
      beta = -copysign(hypot(alpha, xnorm), alpha);
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    if (g == 0 && tid == 0) a.tau[j] = tau;
    __syncthreads();  // every thread has read wv[j] before wv[k] are overwritten below
    // w_k = A_jk + scal d_k
    for (int k = j + 1 + tid; k < n; k += QR_THREADS) wv[k] = __ldcg(&rowj[k]) + scal * wv[k];
    // v over own rows: 0 above j, 1 at j, scaled x below
    for (int i = r0 + tid; i < r1; i += QR_THREADS) {
      double x = 0.0;
      if (i > j) {
        x = col(j)[i] * scal;
        col(j)[i] = x;
      } else if (i == j) {
        x = 1.0;
      }
      vs[i - r0] = x;
    }
    __syncthreads();
    const int i0 = max(r0, j);
    if (j + 1 < n) {
      // column j+1 first: update, keep own rows in xs, squared norm below row j+1
      double* c1 = col(j + 1);
      const double tw1 = tau * wv[j + 1];
      double nacc = 0.0;
      double* rown = rowcopy(j + 1);
      for (int i = r0 + tid; i < r1; i += QR_THREADS) {
        double x = c1[i];
        if (i >= j) {
          x -= tw1 * vs[i - r0];
          c1[i] = x;
        }
        xs[i - r0] = x;
        if (i > j + 1) nacc += x * x;
        if (i == j + 1) rown[j + 1] = x;
      }
      nacc = cta_reduce(nacc, sh + n + 2 * rows_per);  // red scratch after xs
      __syncthreads();
      double* Pn = slot(j + 1);
      if (tid == 0) Pn[n] = nacc;
      // other trailing columns: update and dot with the new column j+1 (rows > j+1)
      for (int k = j + 2 + warp; k < n; k += nwarps) {
        double* ck = col(k);
        const double tw = tau * wv[k];
        double acc = 0.0;
        for (int i = i0 + lane; i < r1; i += 32) {
          const double x = ck[i] - tw * vs[i - r0];
          ck[i] = x;
          if (i > j + 1) acc += xs[i - r0] * x;
          if (i == j + 1) rown[k] = x;
        }
        acc = warp_sum(acc);
        if (lane == 0) Pn[k] = acc;
      }
    }
    if (j >= r0 && j < r1 && tid == 0) col(j)[j] = beta;
  }
}

// Blocked Q (compact WY, LAPACK dlarft/dorg2r order): H_1...H_k = I - V T V^T with V the unit
// lower-trapezoidal reflector block and T upper triangular, so Q = E - V (T V1^T) with
// E = [I_k; 0] and V1 the top k x k block of V.  Two DGEMMs replace k BLAS-2 sweeps.
__global__ void k_wy_prep(const double* A, int m, int k, double* V, double* Q) {
  const size_t total = size_t(m) * k;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const int c = int(e / m), i = int(e - size_t(c) * m);
    V[e] = i < c ? 0.0 : (i == c ? 1.0 : A[e]);
    Q[e] = i == c ? 1.0 : 0.0;
  }
}

// T from S = V^T V (k x k, column-major) and tau: T_jj = tau_j,
// T[0:j, j] = T[0:j, 0:j] (-tau_j S[0:j, j])   (dlarft, direct = F, storev = C)
__global__ void __launch_bounds__(256) k_wy_larft(const double* S, const double* tau, int k, double* T) {
  extern __shared__ double z[];
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) T[e] = 0.0;
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    const double tj = tau[j];
    for (int l = threadIdx.x; l < j; l += blockDim.x) z[l] = -tj * S[size_t(j) * k + l];
    __syncthreads();
    for (int i = threadIdx.x; i < j; i += blockDim.x) {
      double acc = 0.0;
      for (int l = i; l < j; ++l) acc += T[size_t(l) * k + i] * z[l];
      T[size_t(j) * k + i] = acc;
    }
    if (threadIdx.x == 0) T[size_t(j) * k + j] = tj;
    __syncthreads();
  }
}

// The same T by recursive doubling instead of the column recurrence (k <= WY_TREE_MAX): for
// adjacent factored blocks [i0, i0 + b) and [i0 + b, i1),
//   (I - V1 T1 V1^T)(I - V2 T2 V2^T) = I - [V1 V2] [[T1, -T1 S12 T2], [0, T2]] [V1 V2]^T,
// so every level b = 1, 2, 4, ... forms all its off-diagonal blocks T12 = -T11 (S12 T22) in
// parallel (two barriers per level, log2 k levels; tau = 0 needs no special case).  T and the
// W = S12 T22 scratch live in shared memory.
constexpr int WY_TREE_MAX = 112;
__global__ void __launch_bounds__(1024) k_wy_larft_tree(const double* S, const double* tau, int k, double* Tout) {
  extern __shared__ double tsm[];
  double* T = tsm;          // k x k, column-major
  double* W = tsm + k * k;  // S12 T22 at the positions of T12
  const int kk = k * k;
  for (int e = threadIdx.x; e < kk; e += blockDim.x) {
    const int c = e / k, r = e - c * k;
    T[e] = r == c ? tau[c] : 0.0;
  }
  __syncthreads();
  for (int b = 1; b < k; b *= 2) {
    const int b2x = 2 * b;
    for (int e = threadIdx.x; e < kk; e += blockDim.x) {
      const int c = e / k, r = e - c * k;
      const int i0 = (r / b2x) * b2x;
      if (c / b2x * b2x != i0 || r - i0 >= b || c - i0 < b) continue;  // not in this level's T12
      const int j0 = i0 + b;  // W[r][c] = sum_{l = j0}^{c} S[r][l] T[l][c]  (T22 upper)
      double acc = 0.0;
      for (int l = j0; l <= c; ++l) acc = fma(S[size_t(l) * k + r], T[c * k + l], acc);
      W[e] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kk; e += blockDim.x) {
      const int c = e / k, r = e - c * k;
      const int i0 = (r / b2x) * b2x;
      if (c / b2x * b2x != i0 || r - i0 >= b || c - i0 < b) continue;
      double acc = 0.0;  // T12[r][c] = -sum_{l = r}^{i0 + b - 1} T[r][l] W[l][c]  (T11 upper)
      for (int l = r; l < i0 + b; ++l) acc = fma(T[l * k + r], W[c * k + l], acc);
      T[e] = -acc;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < kk; e += blockDim.x) Tout[e] = T[e];
}

// blocked QR helpers: a panel's unit lower-trapezoidal reflectors (rows c0.., ld lda) into V
// (same offsets, ld lda), and the upper triangle of the leading n x n block.
__global__ void k_panel_v(const double* A, int lda, int mp, int w, double* V) {
  const size_t total = size_t(mp) * w;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const int c = int(e / mp), i = int(e - size_t(c) * mp);
    V[size_t(c) * lda + i] = i < c ? 0.0 : (i == c ? 1.0 : A[size_t(c) * lda + i]);
  }
}

__global__ void k_triu(const double* A, int lda, int n, double* R) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    const int c = e / n, i = e - c * n;
    R[e] = i <= c ? A[size_t(c) * lda + i] : 0.0;
  }
}

// R (keep x n) = upper rows of the pivoted factor, un-pivoted: R[:, perm[k]] = Rp[:, k]
__global__ void k_unpivot_r(const double* A, int m, int n, int keep, const int* perm, double* R) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < keep * n; e += gridDim.x * blockDim.x) {
    const int k = e / keep, i = e - k * keep;  // pivoted column k, row i
    R[size_t(perm[k]) * keep + i] = (i <= k) ? A[size_t(k) * m + i] : 0.0;
  }
}

// ---- one-sided Jacobi SVD, single CTA ------------------------------------------------

struct JacobiArgs {
  double* A;  // r x c column-major (r >= c), overwritten by U*Sigma then U
  double* V;  // c x c
  int r, c;
  double* sigma;  // c (sorted desc)
  int* order;     // c scratch
  double* tmp;    // r*c + c*c scratch for the sorted copies
  int max_sweeps;
};

// SMEM: A (r x c) and V (c x c) are staged in shared memory when they fit.  A pair is
// rotated when |a_i . a_j| > sqrt(r) eps |a_i||a_j| (relative orthogonality, as dgesvj) and
// the pair is not negligible against the largest column (|a_i||a_j| > eps^2 max|a_k|^2),
// which keeps round-off-level columns from spinning forever.
template <bool SMEM>
__global__ void __launch_bounds__(1024) k_jacobi(JacobiArgs a) {
  extern __shared__ double js[];
  const int r = a.r, c = a.c;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  __shared__ int rotated;
  __shared__ double colmax;
  double* A = SMEM ? js : a.A;
  double* V = SMEM ? js + size_t(r) * c : a.V;
  if (SMEM)
    for (int e = threadIdx.x; e < r * c; e += blockDim.x) A[e] = a.A[e];
  for (int e = threadIdx.x; e < c * c; e += blockDim.x) V[e] = (e % (c + 1) == 0) ? 1.0 : 0.0;
  const int cc = (c % 2 == 0) ? c : c + 1;  // tournament size (dummy column when odd)
  const double eps = 2.220446049250313e-16;
  const double tol = eps * sqrt(double(r));
  __syncthreads();
  int sweep = 0;
  for (; sweep < a.max_sweeps; ++sweep) {
    if (threadIdx.x == 0) {
      rotated = 0;
      colmax = 0.0;
    }
    __syncthreads();
    for (int k = warp; k < c; k += nwarps) {
      double sacc = 0.0;
      for (int q = lane; q < r; q += 32) sacc += A[size_t(k) * r + q] * A[size_t(k) * r + q];
      sacc = warp_sum(sacc);
      if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(&colmax), __double_as_longlong(sacc));
    }
    __syncthreads();
    const double floor2 = eps * eps * colmax;
    for (int round = 0; round < cc - 1; ++round) {
      // pairs per lane group: 16-lane groups in the shared-memory variant (two pairs per warp at
      // once, half the sequential steps per round), whole warps otherwise (k_jacobi_coop's order)
      constexpr int GS = SMEM ? 16 : 32;
      const int glane = threadIdx.x & (GS - 1), grp = threadIdx.x / GS, ngrp = blockDim.x / GS;
      const unsigned gmask = GS == 32 ? 0xffffffffu : (0xffffu << (threadIdx.x & 16));
      auto gsum = [&](double x) {
        for (int o = GS / 2; o > 0; o >>= 1) x += __shfl_xor_sync(gmask, x, o);
        return x;
      };
      for (int pr = grp; pr < cc / 2; pr += ngrp) {
        auto pos = [&](int q) { return q == 0 ? 0 : 1 + (q - 1 + round) % (cc - 1); };
        int i = pos(pr), j = pos(cc - 1 - pr);
        if (i > j) {
          const int t = i;
          i = j;
          j = t;
        }
        if (j >= c) continue;
        double* ai = A + size_t(i) * r;
        double* aj = A + size_t(j) * r;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int k = glane; k < r; k += GS) {
          const double x = ai[k], y = aj[k];
          al += x * x;
          be += y * y;
          ga += x * y;
        }
        al = gsum(al);
        be = gsum(be);
        ga = gsum(ga);
        const double nab = sqrt(al) * sqrt(be);
        if (ga != 0.0 && fabs(ga) > tol * nab && nab > floor2) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
          for (int k = glane; k < r; k += GS) {
            const double x = ai[k], y = aj[k];
            ai[k] = cs * x - sn * y;
            aj[k] = sn * x + cs * y;
          }
          double* vi = V + size_t(i) * c;
          double* vj = V + size_t(j) * c;
          for (int k = glane; k < c; k += GS) {
            const double x = vi[k], y = vj[k];
            vi[k] = cs * x - sn * y;
            vj[k] = sn * x + cs * y;
          }
          if (glane == 0) rotated = 1;
        }
      }
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  double* sv = a.tmp + size_t(r) * c + size_t(c) * c;
  for (int k = warp; k < c; k += nwarps) {
    double sacc = 0.0;
    for (int q = lane; q < r; q += 32) sacc += A[size_t(k) * r + q] * A[size_t(k) * r + q];
    sacc = warp_sum(sacc);
    if (lane == 0) sv[k] = sqrt(sacc);
  }
  if (threadIdx.x == 0) sv[c] = double(sweep);  // diagnostics: sweeps used
  __syncthreads();
  for (int k = threadIdx.x; k < c; k += blockDim.x) {
    int rank = 0;
    for (int q = 0; q < c; ++q)
      if (sv[q] > sv[k] || (sv[q] == sv[k] && q < k)) ++rank;
    a.order[rank] = k;
  }
  __syncthreads();
  const double* SA = A;
  const double* SV = V;
  if (!SMEM) {  // in-place permutation needs a staging copy
    for (int e = threadIdx.x; e < r * c; e += blockDim.x) a.tmp[e] = A[e];
    for (int e = threadIdx.x; e < c * c; e += blockDim.x) a.tmp[size_t(r) * c + e] = V[e];
    SA = a.tmp;
    SV = a.tmp + size_t(r) * c;
    __syncthreads();
  }
  for (int e = threadIdx.x; e < r * c; e += blockDim.x) {
    const int k = e / r, q = e - k * r;
    const int src = a.order[k];
    const double sg = sv[src];
    a.A[e] = sg > 0.0 ? SA[size_t(src) * r + q] / sg : 0.0;
  }
  for (int e = threadIdx.x; e < c * c; e += blockDim.x) {
    const int k = e / c, q = e - k * c;
    a.V[e] = SV[size_t(a.order[k]) * c + q];
  }
  for (int k = threadIdx.x; k < c; k += blockDim.x) a.sigma[k] = sv[a.order[k]];
}

// One-sided Jacobi for matrices that fit one CTA's shared memory (the corrector's H up to ~110
// columns): the same tournament schedule and stopping rules as k_jacobi, with fewer instructions
// per pair -- the instruction issue of one SM is what bounds this kernel (ncu: ~600 instructions
// per pair-round in k_jacobi).  A GS-lane group owns one pair per round (more rows per lane, so the
// per-pair scalar work is shared by fewer lanes), the pairing advances by conditional subtraction
// instead of a modulo, the rotation test compares squares (ga^2 > tol^2 al be) instead of
// forming sqrt(al) sqrt(be), and cos = rsqrt(1 + t^2).
template <int GS, int RPL>  // r <= GS * RPL (and c <= r), c / 2 * GS <= 512 threads
__global__ void __launch_bounds__(512) k_jacobi_small(JacobiArgs a) {
  extern __shared__ double js[];
  const int r = a.r, c = a.c;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  __shared__ int rotated;
  __shared__ double colmax;
  double* A = js;
  double* V = js + size_t(r) * c;
  for (int e = tid; e < r * c; e += blockDim.x) A[e] = a.A[e];
  for (int e = tid; e < c * c; e += blockDim.x) V[e] = (e % (c + 1) == 0) ? 1.0 : 0.0;
  const int cc = (c % 2 == 0) ? c : c + 1;  // tournament size (dummy column when odd)
  const int m1 = cc - 1;
  const double eps = 2.220446049250313e-16;
  const double tol2 = eps * eps * double(r);
  const int glane = tid & (GS - 1), pr = tid / GS;  // one pair per group
  auto gsum = [&](double x) {  // xor offsets < GS stay inside the group; all 32 lanes take part
#pragma unroll
    for (int o = GS / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
  };
  // tournament positions of this group's pair: pos(q) = q == 0 ? 0 : 1 + (q - 1 + round) % (cc - 1)
  int x1 = pr - 1, x2 = cc - 2 - pr;  // (q - 1) for q = pr and q = cc - 1 - pr, advanced per round
  if (x1 < 0) x1 += m1;               // pr == 0 stays at position 0 (handled below)
  __syncthreads();
  int sweep = 0;
  for (; sweep < a.max_sweeps; ++sweep) {
    if (tid == 0) {
      rotated = 0;
      colmax = 0.0;
    }
    __syncthreads();
    for (int k = warp; k < c; k += nwarps) {
      double sacc = 0.0;
      for (int q = lane; q < r; q += 32) sacc = fma(A[size_t(k) * r + q], A[size_t(k) * r + q], sacc);
      sacc = warp_sum(sacc);
      if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(&colmax), __double_as_longlong(sacc));
    }
    __syncthreads();
    const double floor2 = eps * eps * colmax;
    const double floor4 = floor2 * floor2;
    int y1 = x1, y2 = x2;
    for (int round = 0; round < m1; ++round) {
      // every lane of the warp reaches the shuffles (full-warp masks; a per-group partial mask
      // makes the warp serialise its groups, ncu: BRA.DIV + WARPSYNC on the reductions);
      // inactive groups compute on zeros and store nothing
      int i = pr == 0 ? 0 : 1 + y1, j = 1 + y2;
      if (i > j) {
        const int t = i;
        i = j;
        j = t;
      }
      const bool act = pr < cc / 2 && j < c;
      if (!act) i = j = 0;
      // the pair's rows in registers: all loads issued together, reused by the rotation
      double* ai = A + size_t(i) * r;
      double* aj = A + size_t(j) * r;
      double x[RPL], y[RPL];
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const int k = glane + GS * t;
        x[t] = act && k < r ? ai[k] : 0.0;
        y[t] = act && k < r ? aj[k] : 0.0;
      }
      double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        al = fma(x[t], x[t], al);
        be = fma(y[t], y[t], be);
        ga = fma(x[t], y[t], ga);
      }
      al = gsum(al);
      be = gsum(be);
      ga = gsum(ga);
      const double ab = al * be;
      if (act && ga != 0.0 && ga * ga > tol2 * ab && ab > floor4) {
        const double zeta = (be - al) / (2.0 * ga);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
        const double cs = rsqrt(fma(t, t, 1.0)), sn = cs * t;
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          const int k = glane + GS * u;
          if (k < r) {
            ai[k] = fma(cs, x[u], -sn * y[u]);
            aj[k] = fma(sn, x[u], cs * y[u]);
          }
        }
        double* vi = V + size_t(i) * c;  // V's columns through the same registers
        double* vj = V + size_t(j) * c;
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          const int k = glane + GS * u;
          x[u] = k < c ? vi[k] : 0.0;
          y[u] = k < c ? vj[k] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          const int k = glane + GS * u;
          if (k < c) {
            vi[k] = fma(cs, x[u], -sn * y[u]);
            vj[k] = fma(sn, x[u], cs * y[u]);
          }
        }
        if (glane == 0) rotated = 1;
      }
      if (++y1 == m1) y1 = 0;
      if (++y2 == m1) y2 = 0;
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  double* sv = a.tmp + size_t(r) * c + size_t(c) * c;
  for (int k = warp; k < c; k += nwarps) {
    double sacc = 0.0;
    for (int q = lane; q < r; q += 32) sacc = fma(A[size_t(k) * r + q], A[size_t(k) * r + q], sacc);
    sacc = warp_sum(sacc);
    if (lane == 0) sv[k] = sqrt(sacc);
  }
  if (tid == 0) sv[c] = double(sweep);  // diagnostics: sweeps used
  __syncthreads();
  for (int k = tid; k < c; k += blockDim.x) {
    int rank = 0;
    for (int q = 0; q < c; ++q)
      if (sv[q] > sv[k] || (sv[q] == sv[k] && q < k)) ++rank;
    a.order[rank] = k;
  }
  __syncthreads();
  for (int e = tid; e < r * c; e += blockDim.x) {
    const int k = e / r, q = e - k * r;
    const int src = a.order[k];
    const double sg = sv[src];
    a.A[e] = sg > 0.0 ? A[size_t(src) * r + q] / sg : 0.0;
  }
  for (int e = tid; e < c * c; e += blockDim.x) {
    const int k = e / c, q = e - k * c;
    a.V[e] = V[size_t(a.order[k]) * c + q];
  }
  for (int k = tid; k < c; k += blockDim.x) a.sigma[k] = sv[a.order[k]];
}

// One-sided Jacobi on a thread-block cluster (JC_CS CTAs): the single-SM kernels above are bound
// by one SM's shared-memory bandwidth -- every round streams all of A and V through it.  Here the
// ROWS of A and V are split over the cluster (rotations act on columns, so rows are independent):
// each round every CTA forms its partial (a_i.a_i, a_j.a_j, a_i.a_j) of every pair over its own
// rows and pushes them into every rank's shared memory with st.async (bytes completed on the
// receiver's mbarrier: no cluster barrier per round -- a cluster barrier's release waits for the
// remote stores, ncu: ERRBAR 31 % of stall samples); then every CTA sums the partials of every
// pair in the same fixed rank order, takes the same decision and applies the rotation to its own
// rows.  Same tournament schedule and stopping rules as k_jacobi_small; deterministic.
constexpr int JC_CS = 8;

template <int JC_GS>  // lanes per pair
__global__ void __launch_bounds__(1024) k_jacobi_cluster(JacobiArgs a) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ double jc[];
  const int q = int(cluster.block_rank());
  const int r = a.r, c = a.c;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int ra0 = q * r / JC_CS, na = (q + 1) * r / JC_CS - ra0;  // own rows of A
  const int rv0 = q * c / JC_CS, nv = (q + 1) * c / JC_CS - rv0;  // own rows of V
  const int cc = (c % 2 == 0) ? c : c + 1, m1 = cc - 1, pairs = cc / 2;
  // the exchanged buffers first: map_shared_rank maps the same offset in every CTA, and the row
  // counts (hence the A/V tile sizes) differ between CTAs
  double* gath = jc;                        // [2][CS][pairs][4]: partials pushed by every rank
  double* stg = gath + 2 * JC_CS * 4 * pairs;  // [2][pairs][4]: this rank's partials, staged
  double* cn = stg + 2 * 4 * pairs;         // [2][c]: per-column partial norms
  double* sv = cn + 2 * c;                  // c
  int* order = reinterpret_cast<int*>(sv + c);  // c (c / 2 doubles)
  double* Ao = sv + c + (c + 1) / 2;        // c columns x na rows
  double* Vo = Ao + size_t(c) * na;         // c columns x nv rows
  __shared__ int any_rot, nrot;
  __shared__ double s_colmax;
  __shared__ __align__(8) unsigned long long bars[2];  // one mbarrier per exchange buffer
  const unsigned bar0 = smem_addr(&bars[0]);
  const unsigned round_bytes = unsigned(JC_CS * pairs * 4 * sizeof(double));
  if (tid == 0) {
    mbar_init(bar0, 1);
    mbar_init(bar0 + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int e = tid; e < c * na; e += blockDim.x) {
    const int k = e / na, t = e - k * na;
    Ao[e] = a.A[size_t(k) * r + ra0 + t];
  }
  for (int e = tid; e < c * nv; e += blockDim.x) {
    const int k = e / nv, t = e - k * nv;
    Vo[e] = (rv0 + t == k) ? 1.0 : 0.0;
  }
  const double eps = 2.220446049250313e-16;
  const double tol2 = eps * eps * double(r);
  const int glane = tid & (JC_GS - 1), pr = tid / JC_GS;
  auto gsum = [&](double x) {  // xor offsets < GS stay inside the group; all 32 lanes take part
#pragma unroll
    for (int o = JC_GS / 2; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
  };
  long long ph[5] = {0, 0, 0, 0, 0};  // diagnostics (rank 0, thread 0 written at the end)
  int it = 0;  // parity of the column-norm buffers, advanced at every column-norm exchange
  int ex = 0;  // pair-partial exchanges so far (buffer and mbarrier phase)
  // column norms^2 of A over the cluster -> sv (identical in every CTA)
  auto column_norms2 = [&]() {
    double* pb = cn + (it & 1) * c;
    for (int k = warp; k < c; k += nwarps) {
      double acc = 0.0;
      for (int t = lane; t < na; t += 32) acc = fma(Ao[size_t(k) * na + t], Ao[size_t(k) * na + t], acc);
      acc = warp_sum(acc);
      if (lane == 0) pb[k] = acc;
    }
    cluster.sync();
    for (int k = tid; k < c; k += blockDim.x) {
      double acc = 0.0;
      for (int o = 0; o < JC_CS; ++o) acc += cluster.map_shared_rank(pb, o)[k];
      sv[k] = acc;
    }
    ++it;
    __syncthreads();
  };
  int x1 = pr - 1, x2 = cc - 2 - pr;
  if (x1 < 0) x1 += m1;
  cluster.sync();  // mbarriers initialised before any rank sends
  int sweep = 0;
  for (; sweep < a.max_sweeps; ++sweep) {
    column_norms2();
    if (warp == 0) {
      double mx = 0.0;
      for (int k = lane; k < c; k += 32) mx = fmax(mx, sv[k]);
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) {
        s_colmax = mx;
        any_rot = 0;
        nrot = 0;
      }
    }
    __syncthreads();
    const double floor2 = eps * eps * s_colmax;
    const double floor4 = floor2 * floor2;
    int y1 = x1, y2 = x2;
    for (int round = 0; round < m1; ++round, ++ex) {
      // exchange ex: buffer ex & 1, mbarrier phase (ex >> 1) & 1 (no cluster barrier per round:
      // a rank sends round ex + 2 into this buffer only after receiving this rank's round ex + 1
      // partials, which are sent after this round's reads)
      double* gb = gath + (ex & 1) * JC_CS * 4 * pairs;
      const unsigned bar = bar0 + 8u * unsigned(ex & 1);
      const long long tc0 = clock64();
      if (tid == 0) mbar_expect(bar, round_bytes);
      int i = 0, j = 0;
      bool act = false;
      if (pr < pairs) {
        i = pr == 0 ? 0 : 1 + y1;
        j = 1 + y2;
        if (i > j) {
          const int t = i;
          i = j;
          j = t;
        }
        act = j < c;
      }
      double* ai = Ao + size_t(i) * na;
      double* aj = Ao + size_t(j) * na;
      // all lanes reach the shuffles (full-warp masks); inactive groups sum zeros, send nothing
      double al = 0.0, be = 0.0, ga = 0.0;
      if (act)
        for (int t = glane; t < na; t += JC_GS) {
          const double x = ai[t], y = aj[t];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
      al = gsum(al);
      be = gsum(be);
      ga = gsum(ga);
      // all-gather by push: the partials of all pairs are staged locally, then thread t < CS
      // sends the block to rank t with ONE bulk copy completing on rank t's mbarrier (per-pair
      // st.async made every CTA's mbarrier absorb CS x pairs transaction updates per round)
      double* sg = stg + (ex & 1) * 4 * pairs;
      if (act && glane == 0) {
        sg[4 * pr] = al;
        sg[4 * pr + 1] = be;
        sg[4 * pr + 2] = ga;
      }
      __syncthreads();
      if (tid < JC_CS) {
        fence_proxy_async_smem();
        bulk_to_peer(cluster_map(smem_addr(gb + size_t(q) * pairs * 4), tid), smem_addr(sg),
                     unsigned(pairs * 4 * sizeof(double)), cluster_map(bar, tid));
      }
      const long long tc1 = clock64();
      mbar_wait(bar, unsigned(ex >> 1) & 1u);
      const long long tc2 = clock64();
      {
        // lane l sums ranks l, l + GS, ... (local shared memory), then the group tree: the same
        // fixed order in every CTA, so every CTA takes the same decision for every pair
        double s0 = 0.0, s1 = 0.0, s2 = 0.0;
        if (act)
#pragma unroll
          for (int o = glane; o < JC_CS; o += JC_GS) {
            const double* sp = gb + (size_t(o) * pairs + pr) * 4;
            s0 += sp[0];
            s1 += sp[1];
            s2 += sp[2];
          }
        const double al2 = gsum(s0), be2 = gsum(s1), ga2 = gsum(s2);
        const double ab = al2 * be2;
        if (act && ga2 != 0.0 && ga2 * ga2 > tol2 * ab && ab > floor4) {
          const double zeta = (be2 - al2) / (2.0 * ga2);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
          const double cs = rsqrt(fma(t, t, 1.0)), sn = cs * t;
          for (int u = glane; u < na; u += JC_GS) {
            const double x = ai[u], y = aj[u];
            ai[u] = fma(cs, x, -sn * y);
            aj[u] = fma(sn, x, cs * y);
          }
          double* vi = Vo + size_t(i) * nv;
          double* vj = Vo + size_t(j) * nv;
          for (int u = glane; u < nv; u += JC_GS) {
            const double x = vi[u], y = vj[u];
            vi[u] = fma(cs, x, -sn * y);
            vj[u] = fma(sn, x, cs * y);
          }
          if (glane == 0) {
            any_rot = 1;
            atomicAdd(&nrot, 1);
          }
        }
      }
      const long long tc3 = clock64();
      if (++y1 == m1) y1 = 0;
      if (++y2 == m1) y2 = 0;
      __syncthreads();
      const long long tc4 = clock64();
      ph[0] += tc1 - tc0;  // diagnostics: cycles per phase, summed over rounds (registers)
      ph[1] += tc2 - tc1;
      ph[2] += tc3 - tc2;
      ph[3] += tc4 - tc3;
      ++ph[4];
    }
    if (q == 0 && tid == 0 && sweep < 16) a.tmp[size_t(r) * c + size_t(c) * c + c + 1 + sweep] = double(nrot);
    if (!any_rot) break;
  }
  column_norms2();
  for (int k = tid; k < c; k += blockDim.x) sv[k] = sqrt(sv[k]);
  __syncthreads();
  for (int k = tid; k < c; k += blockDim.x) {
    int rank = 0;
    for (int o = 0; o < c; ++o)
      if (sv[o] > sv[k] || (sv[o] == sv[k] && o < k)) ++rank;
    order[rank] = k;
  }
  __syncthreads();
  for (int e = tid; e < c * na; e += blockDim.x) {
    const int k = e / na, t = e - k * na;
    const int src = order[k];
    const double sg = sv[src];
    a.A[size_t(k) * r + ra0 + t] = sg > 0.0 ? Ao[size_t(src) * na + t] / sg : 0.0;
  }
  for (int e = tid; e < c * nv; e += blockDim.x) {
    const int k = e / nv, t = e - k * nv;
    a.V[size_t(k) * c + rv0 + t] = Vo[size_t(order[k]) * nv + t];
  }
  if (q == 0) {
    for (int k = tid; k < c; k += blockDim.x) a.sigma[k] = sv[order[k]];
    if (tid == 0) {  // diagnostics
      double* dg = a.tmp + size_t(r) * c + size_t(c) * c + c;
      dg[0] = double(sweep);
      for (int k = 0; k < 5; ++k) dg[17 + k] = double(ph[k]);
    }
  }
  cluster.sync();  // no CTA leaves while another may still read its shared memory
}

// Multi-CTA one-sided Jacobi for matrices that do not fit one CTA's shared memory: the same
// tournament schedule and per-pair arithmetic as k_jacobi (warp-strided sums, xor-shuffle
// reduction, same rotation and stopping rules), so the result is bitwise the one k_jacobi<false>
// computes; the c/2 pairs of a round are spread over all warps of the grid and a grid barrier
// separates rounds.  A and V live in global memory (L2) and are read with __ldcg: another SM
// may have rotated a column since this SM last cached it.  `ctl` (global): [0..1] colmax bits,
// [2..3] rotated flags (double-buffered by sweep parity), [4] sweeps used.
__global__ void __launch_bounds__(256) k_jacobi_coop(JacobiArgs a, unsigned long long* ctl) {
  cg::grid_group grid = cg::this_grid();
  const int r = a.r, c = a.c;
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int gw = blockIdx.x * nw + (threadIdx.x >> 5), tw = gridDim.x * nw;
  double* A = a.A;
  double* V = a.V;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < size_t(c) * c; e += size_t(gridDim.x) * blockDim.x)
    V[e] = (e % (c + 1) == 0) ? 1.0 : 0.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) ctl[0] = ctl[1] = ctl[2] = ctl[3] = 0ull;
  const int cc = (c % 2 == 0) ? c : c + 1;
  const double eps = 2.220446049250313e-16;
  const double tol = eps * sqrt(double(r));
  grid.sync();
  int sweep = 0;
  for (; sweep < a.max_sweeps; ++sweep) {
    const int par = sweep & 1;
    for (int k = gw; k < c; k += tw) {
      double sacc = 0.0;
      for (int q = lane; q < r; q += 32) {
        const double x = __ldcg(&A[size_t(k) * r + q]);
        sacc += x * x;
      }
      sacc = warp_sum(sacc);
      if (lane == 0) atomicMax(&ctl[par], static_cast<unsigned long long>(__double_as_longlong(sacc)));
    }
    grid.sync();
    // every block has finished sweep - 1 (incl. reading its rotated flag): clear its slots,
    // which sweep + 1 reuses
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl[par ^ 1] = ctl[2 + (par ^ 1)] = 0ull;
    const double floor2 = eps * eps * __longlong_as_double(static_cast<long long>(__ldcg(&ctl[par])));
    for (int round = 0; round < cc - 1; ++round) {
      for (int pr = gw; pr < cc / 2; pr += tw) {
        auto pos = [&](int q) { return q == 0 ? 0 : 1 + (q - 1 + round) % (cc - 1); };
        int i = pos(pr), j = pos(cc - 1 - pr);
        if (i > j) {
          const int t = i;
          i = j;
          j = t;
        }
        if (j >= c) continue;
        double* ai = A + size_t(i) * r;
        double* aj = A + size_t(j) * r;
        double al = 0.0, be = 0.0, ga = 0.0;
        // loads 4 rows ahead (L2 latency), accumulation in k order as k_jacobi (bitwise equal)
        int k = lane;
        for (; k + 96 < r; k += 128) {
          double x[4], y[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            x[u] = __ldcg(&ai[k + 32 * u]);
            y[u] = __ldcg(&aj[k + 32 * u]);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            al += x[u] * x[u];
            be += y[u] * y[u];
            ga += x[u] * y[u];
          }
        }
        for (; k < r; k += 32) {
          const double x = __ldcg(&ai[k]), y = __ldcg(&aj[k]);
          al += x * x;
          be += y * y;
          ga += x * y;
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        const double nab = sqrt(al) * sqrt(be);
        if (ga != 0.0 && fabs(ga) > tol * nab && nab > floor2) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
          auto rotate = [&](double* pi, double* pj, int len) {
            int q = lane;
            for (; q + 96 < len; q += 128) {
              double x[4], y[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                x[u] = __ldcg(&pi[q + 32 * u]);
                y[u] = __ldcg(&pj[q + 32 * u]);
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                __stcg(&pi[q + 32 * u], cs * x[u] - sn * y[u]);
                __stcg(&pj[q + 32 * u], sn * x[u] + cs * y[u]);
              }
            }
            for (; q < len; q += 32) {
              const double x = __ldcg(&pi[q]), y = __ldcg(&pj[q]);
              __stcg(&pi[q], cs * x - sn * y);
              __stcg(&pj[q], sn * x + cs * y);
            }
          };
          rotate(ai, aj, r);
          rotate(V + size_t(i) * c, V + size_t(j) * c, c);
          if (lane == 0) ctl[2 + par] = 1ull;
        }
      }
      grid.sync();
    }
    if (__ldcg(&ctl[2 + par]) == 0ull) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ctl[4] = static_cast<unsigned long long>(sweep);
}

// Epilogue of the multi-CTA path (single CTA): singular values = column norms, descending
// order with index tie-break, U = A P / sigma, V P — as k_jacobi's tail.
__global__ void __launch_bounds__(1024) k_jacobi_finish(JacobiArgs a, const unsigned long long* ctl) {
  const int r = a.r, c = a.c;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  double* sv = a.tmp + size_t(r) * c + size_t(c) * c;
  for (int k = warp; k < c; k += nwarps) {
    double sacc = 0.0;
    for (int q = lane; q < r; q += 32) sacc += a.A[size_t(k) * r + q] * a.A[size_t(k) * r + q];
    sacc = warp_sum(sacc);
    if (lane == 0) sv[k] = sqrt(sacc);
  }
  if (threadIdx.x == 0) sv[c] = double(ctl[4]);
  __syncthreads();
  for (int k = threadIdx.x; k < c; k += blockDim.x) {
    int rank = 0;
    for (int q = 0; q < c; ++q)
      if (sv[q] > sv[k] || (sv[q] == sv[k] && q < k)) ++rank;
    a.order[rank] = k;
  }
  for (int e = threadIdx.x; e < r * c; e += blockDim.x) a.tmp[e] = a.A[e];
  for (int e = threadIdx.x; e < c * c; e += blockDim.x) a.tmp[size_t(r) * c + e] = a.V[e];
  __syncthreads();
  const double* SA = a.tmp;
  const double* SV = a.tmp + size_t(r) * c;
  for (int e = threadIdx.x; e < r * c; e += blockDim.x) {
    const int k = e / r, q = e - k * r;
    const int src = a.order[k];
    const double sg = sv[src];
    a.A[e] = sg > 0.0 ? SA[size_t(src) * r + q] / sg : 0.0;
  }
  for (int e = threadIdx.x; e < c * c; e += blockDim.x) {
    const int k = e / c, q = e - k * c;
    a.V[e] = SV[size_t(a.order[k]) * c + q];
  }
  for (int k = threadIdx.x; k < c; k += blockDim.x) a.sigma[k] = sv[a.order[k]];
}

__global__ void k_transpose(const double* in, int rows, int cols, double* out) {
  // in: rows x cols (col-major) -> out: cols x rows
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += gridDim.x * blockDim.x) {
    const int j = e / rows, i = e - j * rows;
    out[size_t(i) * cols + j] = in[e];
  }
}

__global__ void __launch_bounds__(256) k_fix_signs(double* X, double* Y, int rows) {
  const int j = blockIdx.x;
  double* x = X + size_t(j) * rows;
  double* y = Y + size_t(j) * rows;
  __shared__ double bv[256];
  __shared__ int bi[256];
  double best = -1.0;
  int idx = 0;
  for (int i = threadIdx.x; i < rows; i += 256) {
    const double a = fabs(x[i]);
    if (a > best) {  // strictly greater: first maximum within the thread's stride
      best = a;
      idx = i;
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = idx;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double o = bv[threadIdx.x + s];
      const int oi = bi[threadIdx.x + s];
      if (o > bv[threadIdx.x] || (o == bv[threadIdx.x] && oi < bi[threadIdx.x])) {
        bv[threadIdx.x] = o;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  const bool flip = rows > 0 && x[bi[0]] < 0.0;
  __syncthreads();
  if (flip)
    for (int i = threadIdx.x; i < rows; i += 256) {
      x[i] = -x[i];
      y[i] = -y[i];
    }
}

// H = [UF; RF] [VG; RG]^T + diag(S, 0): assembled blocks (col-major)
__global__ void k_stack_rows(const double* top, int rt, const double* bot, int rb, int cols, double* out) {
  const int rows = rt + rb;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += gridDim.x * blockDim.x) {
    const int j = e / rows, i = e - j * rows;
    out[e] = i < rt ? top[size_t(j) * rt + i] : bot[size_t(j) * rb + (i - rt)];
  }
}

__global__ void k_add_diag(double* H, int ld, const double* s, int r) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < r; i += gridDim.x * blockDim.x)
    H[size_t(i) * ld + i] += s[i];
}

// deterministic two-stage sum of squares: fixed grid, per-block partials, one final block
__global__ void __launch_bounds__(256) k_sumsq_part(const double* x, size_t n, double* part) {
  __shared__ double red[256];
  double s = 0.0;
  for (size_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += size_t(gridDim.x) * 256) s += x[i] * x[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void __launch_bounds__(256) k_sum_final(const double* part, int np, double* out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += 256) s += part[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

double dev_sumsq(ptb_context* ctx, const double* x, size_t n, DeviceBuffer& scratch) {
  constexpr int NP = 296;  // fixed partial count (2 x 148 SMs): deterministic for a given n
  double* d = static_cast<double*>(scratch.get((NP + 1) * sizeof(double)));
  k_sumsq_part<<<NP, 256, 0, ctx->stream>>>(x, n, d + 1);
  PTB_LAUNCH_CHECK(ctx);
  k_sum_final<<<1, 256, 0, ctx->stream>>>(d + 1, NP, d);
  PTB_LAUNCH_CHECK(ctx);
  double h = 0.0;
  PTB_CUDA_CHECK(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  PTB_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  return h;
}

int qr_grid(ptb_context* ctx, int m, size_t smem, const void* kern, int rows_per_cta = 512) {
  int per_sm = 0;
  PTB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, QR_THREADS, smem));
  const int cap = std::max(1, per_sm) * ctx->num_sms;
  const int want = std::max(1, (m + rows_per_cta - 1) / rows_per_cta);
  return std::min({cap, want, ctx->num_sms});
}

}  // namespace

ProcWork::ProcWork(ptb_context* c) : ctx(c) {}
ProcWork::~ProcWork() {
  for (auto& b : buf) b.release();
  for (DeviceBuffer* b : {&QF, &RF, &QG, &RG, &Uh, &Vh, &PQ, &PR, &PU, &SX, &SY, &BA, &BV, &BT, &BR, &BQ2})
    b->release();
  for (auto& b : TS) b.release();
  for (auto& b : TX) b.release();
  for (auto& b : TS2) b.release();
  for (auto& b : TX2) b.release();
  for (auto& b : PA) b.release();
  for (auto& b : PB) b.release();
  BQ2b.release();
}

DevCorrector::~DevCorrector() {
  X.release();
  Y.release();
  Sd.release();
}

void DevCorrector::assign(int rows_, int rank_, const std::vector<double>& s, double tol_) {
  rows = rows_;
  rank = rank_;
  S = s;
  tol = tol_;
  double* d = static_cast<double*>(Sd.get(std::max<size_t>(1, S.size()) * sizeof(double)));
  if (!S.empty())
    PTB_CUDA_CHECK(cudaMemcpy(d, S.data(), S.size() * sizeof(double), cudaMemcpyHostToDevice));
}

void wy_larft(ptb_context* ctx, cudaStream_t st, const double* S, const double* tau, int k, double* T) {
  if (k <= WY_TREE_MAX) {
    const size_t smem = size_t(2) * k * k * sizeof(double);
    PTB_CUDA_CHECK(cudaFuncSetAttribute(k_wy_larft_tree, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    k_wy_larft_tree<<<1, 1024, smem, st>>>(S, tau, k, T);
  } else {
    k_wy_larft<<<1, 256, size_t(k) * sizeof(double), st>>>(S, tau, k, T);
  }
  PTB_LAUNCH_CHECK(ctx);
}

// ---- TSQR: tall-skinny QR as a reduction tree (n <= TS_MAXN) ------------------------------
// Level l splits its m_l rows into nb_l leaves of <= TS_ROWS rows (sizes differ by at most one,
// so every leaf has >= TS_ROWS / 2 >= n rows); each leaf is an unpivoted Householder QR in one
// CTA's shared memory (no grid barrier), its n x n R goes into the next level's stack
// (nb_l n rows).  When the stack fits one leaf, its column-pivoted QR (k_qrcp_small, the
// reference's keep rule) gives the pivots, keep and R -- column norms are invariant under the
// leaves' orthogonal factors, so these are A's own pivoted-QR decisions up to rounding, as in
// the blocked route -- and the thin Q is assembled top-down, each leaf applying its reflectors
// to its n-row slice of the level above (padded with zeros to the leaf's rows).  Leaves are
// k_qr_reg<.., TS = true> (below), the down-sweep k_tsqr_apply4.
constexpr int TS_ROWS = 256, TS_MAXN = 64;

__device__ __forceinline__ int ts_row0(int i, int m, int nb) { return int((long long)i * m / nb); }

// ---- register-resident Householder QR of a small block (one CTA) -------------------------
// Column k lives in the registers of warp k % QRR_WARPS (slot k / QRR_WARPS); lane l holds rows
// l + 32 u.  Per step j: every warp picks the same pivot (PIVOT: largest remaining squared norm,
// first position on ties, positions swapped as dgeqp3 swaps columns -- each warp keeps its own
// copy of the position table), the pivot's owner forms the reflector (dlarfg: beta, tau, scal)
// and publishes the column through shared memory, then every warp applies H_j to its own
// columns from registers and (PIVOT) recomputes their exact squared norms below row j.  Two
// barriers per step; no shared-memory traffic for the trailing matrix.  Keep rule, outputs and
// layout as k_qrcp_small (TS = false: pivoted columns in place, R above and beta on the
// diagonal, scaled reflectors below; TS = true: a TSQR leaf -- reflectors to V, R to the stack).
constexpr int QRR_THREADS = 512, QRR_WARPS = QRR_THREADS / 32;

constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }

// C per-lane partial sums -> the C warp totals in every lane, by a transposed butterfly: the first
// log2 C levels exchange half of the values still held (C - 1 double shuffles in all), the rest
// reduce one value, then the C totals are broadcast -- 10 double shuffles for C = 4 instead of 20.
// Column c ends in lanes [c 32 / C, (c + 1) 32 / C).  Fixed order: deterministic.
template <int C>
__device__ __forceinline__ void warp_allsum(double (&v)[C]) {
  constexpr int L = ilog2(C);
  static_assert((1 << L) == C && C <= 32, "power of two");
  const int lane = threadIdx.x & 31;
  double t[C];
#pragma unroll
  for (int c = 0; c < C; ++c) t[c] = v[c];
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const int o = 16 >> l, half = C >> (l + 1);
    const bool hi = lane & o;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const double keep = hi ? t[half + i] : t[i], give = hi ? t[i] : t[half + i];
      t[i] = keep + __shfl_xor_sync(0xffffffffu, give, o);
    }
  }
#pragma unroll
  for (int o = 16 >> L; o > 0; o >>= 1) t[0] += __shfl_xor_sync(0xffffffffu, t[0], o);
#pragma unroll
  for (int c = 0; c < C; ++c) v[c] = __shfl_sync(0xffffffffu, t[0], c * (32 / C));
}

struct QrRegArgs {
  const double* A;  // input columns, ld lda; TS: this leaf's rows start at ts_row0(blockIdx.x)
  int lda, m, n, nb;
  int pivot;
  double drop_tol;
  double* out;  // !TS: pivoted factor, m x n, ld m
  double* V;    // TS: reflectors, ld ldv (rows of the leaf)
  int ldv;
  double* R;    // TS: stack, ld ldr (leaf i at rows i n)
  int ldr;
  double* tau;  // !TS: n; TS: nb x n
  int* perm;
  int* keep_out;
  double* beta_out;
};

// explicit predicated selects (selp): unlike a ternary over an unrolled slot loop, the front end
// cannot fold these into a dynamically indexed register array
__device__ __forceinline__ double selp(bool c, double a, double b) {
  double r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %3, 0;\n\tselp.f64 %0, %1, %2, q;\n\t}"
      : "=d"(r) : "d"(a), "d"(b), "r"(int(c)));
  return r;
}
__device__ __forceinline__ int selp(bool c, int a, int b) {
  int r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %3, 0;\n\tselp.s32 %0, %1, %2, q;\n\t}"
      : "=r"(r) : "r"(a), "r"(b), "r"(int(c)));
  return r;
}

// Two independent matrices per launch (update_svd's F and G): TS: blockIdx.y, else blockIdx.x
// selects the argument set.
template <int CPW, int RPL, bool PIVOT, bool TS>
__global__ void __launch_bounds__(QRR_THREADS) k_qr_reg(const QrRegArgs a0, const QrRegArgs a1) {
  pdl_wait();  // PDL launches: inputs come from the previous TSQR level
  pdl_trigger();
  const QrRegArgs& a = (TS ? blockIdx.y : blockIdx.x) == 0 ? a0 : a1;
  constexpr int NMAX = CPW * QRR_WARPS, MMAX = 32 * RPL;
  __shared__ double cbuf[MMAX];
  __shared__ double nrm[2][NMAX];
  __shared__ double betas[NMAX], scals[NMAX];
  __shared__ int exps[NMAX];
  __shared__ double s_sc[3];
  __shared__ int s_ex;
  __shared__ int posc[PIVOT ? QRR_WARPS : 1][PIVOT ? NMAX : 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = a.n;
  int r0 = 0, m = a.m;
  if (TS) {  // leaf blockIdx.x of matrix blockIdx.y
    r0 = ts_row0(blockIdx.x, a.m, a.nb);
    m = ts_row0(blockIdx.x + 1, a.m, a.nb) - r0;
  }
  double x[CPW][RPL];
  int estep[CPW];  // step at which the column was eliminated (-1: not yet)
#pragma unroll
  for (int s = 0; s < CPW; ++s) {
    const int k = warp + QRR_WARPS * s;
    estep[s] = -1;
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
      const int r = lane + 32 * u;
      x[s][u] = (k < n && r < m) ? a.A[size_t(k) * a.lda + r0 + r] : 0.0;
    }
    if (PIVOT && k < n) {
      double acc = 0.0;
#pragma unroll
      for (int u = 0; u < RPL; ++u) acc = fma(x[s][u], x[s][u], acc);
      acc = warp_sum(acc);
      if (lane == 0) nrm[0][k] = acc;
    }
  }
  if (PIVOT)
    for (int q = lane; q < n; q += 32) posc[warp][q] = q;
  __syncthreads();
  const int steps = min(m, n);
  int keep = steps;
  for (int j = 0; j < steps; ++j) {
    const int par = j & 1;
    int p = j;
    if (PIVOT) {
      double best = -1.0;
      int bpos = n;
      for (int q = j + lane; q < n; q += 32) {
        const double v = nrm[par][posc[warp][q]];
        if (v > best) {
          best = v;
          bpos = q;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bpos, o);
        if (ob > best || (ob == best && oi < bpos)) {
          best = ob;
          bpos = oi;
        }
      }
      p = posc[warp][bpos];
      __syncwarp();
      if (lane == 0) {
        posc[warp][bpos] = posc[warp][j];
        posc[warp][j] = p;
      }
      __syncwarp();
    }
    if (warp == p % QRR_WARPS) {  // the pivot's owner: dlarfg, publish the column
      // the pivot's slot is dynamic: gather it with explicit selects (an indexed read would move
      // the whole register tile to local memory)
      const int sp = p / QRR_WARPS;
      double cv[RPL], xs = 0.0;
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        double c = x[0][u];
#pragma unroll
        for (int s = 1; s < CPW; ++s) c = selp(sp == s, x[s][u], c);
        cv[u] = c;
        if (lane + 32 * u > j) xs = fma(c, c, xs);
      }
#pragma unroll
      for (int s = 0; s < CPW; ++s) estep[s] = selp(sp == s, j, estep[s]);
      xs = warp_sum(xs);
      // dlarfg on the column scaled by 2^-ex (max |entry| in [1, 2)) when its squares may have
      // underflowed: a TSQR leaf can hold a column of tiny entries (snapshot rows far from the
      // wave, down to denormals); an unscaled norm then yields a non-orthogonal reflector,
      // harmless for the tiny leaf data but not for the O(1) rows the down-sweep applies it to.
      // Above 2^-600 every underflowed square is below 2^-200 of the norm: no scaling (ex = 0).
      int ex = 0;
      if (xs < 0x1p-600) {  // warp-uniform (xs is the warp total)
        double amax = 0.0;
#pragma unroll
        for (int u = 0; u < RPL; ++u)
          if (lane + 32 * u >= j) amax = fmax(amax, fabs(cv[u]));
        for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        ex = amax > 0.0 ? ilogb(amax) : 0;
        xs = 0.0;
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          cv[u] = scalbn(cv[u], -ex);
          if (lane + 32 * u > j) xs = fma(cv[u], cv[u], xs);
        }
        xs = warp_sum(xs);
      }
      double alc = 0.0;
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        if (u == j / 32) alc = cv[u];
        cbuf[lane + 32 * u] = cv[u];
      }
      const double al = __shfl_sync(0xffffffffu, alc, j & 31);
      if (lane == 0) {
        double beta, tau, scal;
        if (xs == 0.0) {
          beta = al;
          tau = 0.0;
          scal = 0.0;
        } else {
          beta = -copysign(sqrt(fma(al, al, xs)), al);
          tau = (beta - al) / beta;
          scal = 1.0 / (al - beta);
        }
        s_sc[0] = scalbn(beta, ex);  // R_jj in the column's own scale
        s_sc[1] = tau;
        s_sc[2] = scal;  // applies to the SCALED column (cbuf)
        s_ex = ex;
      }
    }
    __syncthreads();
    const double beta = s_sc[0], tau = s_sc[1], scal = s_sc[2];
    if (fabs(beta) <= a.drop_tol) {  // first pivot at or below the guard: keep = j
      if (tid == 0 && a.beta_out) a.beta_out[j] = fabs(beta);
      keep = j;
#pragma unroll
      for (int s = 0; s < CPW; ++s) estep[s] = selp(estep[s] == j, -1, estep[s]);
      break;
    }
    if (tid == 0) {
      betas[j] = beta;
      scals[j] = scal;  // reflector of the unscaled column: v = (x 2^-ex) scal
      exps[j] = s_ex;
      if (TS) a.tau[size_t(blockIdx.x) * n + j] = tau;
      else a.tau[j] = tau;
      if (!TS && a.beta_out) a.beta_out[j] = fabs(beta);
    }
    double v[RPL];
#pragma unroll
    for (int u = 0; u < RPL; ++u) {
      const int r = lane + 32 * u;
      v[u] = r > j ? cbuf[r] * scal : (r == j ? 1.0 : 0.0);
    }
    double w[CPW];
#pragma unroll
    for (int s = 0; s < CPW; ++s) {
      double acc = 0.0;
#pragma unroll
      for (int u = 0; u < RPL; ++u) acc = fma(v[u], x[s][u], acc);
      w[s] = acc;
    }
    warp_allsum<CPW>(w);
    double nn[CPW];
#pragma unroll
    for (int s = 0; s < CPW; ++s) {
      const int k = warp + QRR_WARPS * s;
      nn[s] = 0.0;
      if (k >= n || estep[s] >= 0) continue;  // eliminated columns keep their R entries
      const double tw = tau * w[s];
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        const int r = lane + 32 * u;
        x[s][u] = fma(-tw, v[u], x[s][u]);
        if (PIVOT && r > j) nn[s] = fma(x[s][u], x[s][u], nn[s]);
      }
    }
    if (PIVOT) {
      warp_allsum<CPW>(nn);
      if (lane == 0)
#pragma unroll
        for (int s = 0; s < CPW; ++s) {
          const int k = warp + QRR_WARPS * s;
          if (k < n) nrm[par ^ 1][k] = nn[s];
        }
    }
    __syncthreads();
  }
  // outputs: each warp writes its own columns
#pragma unroll
  for (int s = 0; s < CPW; ++s) {
    const int k = warp + QRR_WARPS * s;
    if (k >= n) continue;
    int pos = k;
    if (PIVOT)
      for (int q = 0; q < n; ++q)
        if (posc[warp][q] == k) pos = q;
    const int e = estep[s];
    if (TS) {
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        const int r = lane + 32 * u;
        if (r >= m) continue;
        if (r > k) a.V[size_t(k) * a.ldv + r0 + r] = scalbn(x[s][u], -exps[k]) * scals[k];
        if (r < n) a.R[size_t(k) * a.ldr + size_t(blockIdx.x) * n + r] = r < k ? x[s][u] : (r == k ? betas[k] : 0.0);
      }
    } else {
#pragma unroll
      for (int u = 0; u < RPL; ++u) {
        const int r = lane + 32 * u;
        if (r >= m) continue;
        double val = x[s][u];
        if (e >= 0 && r == e) val = betas[e];
        else if (e >= 0 && r > e) val = scalbn(x[s][u], -exps[e]) * scals[e];
        a.out[size_t(pos) * m + r] = val;
      }
      if (lane == 0) a.perm[pos] = k;
    }
  }
  if (!TS && tid == 0) *a.keep_out = keep;
}

// Xout[leaf rows, :] = H_0 ... H_{n-1} [Xin[i n : i n + n, :]; 0] -- one warp per four columns of
// X held in registers (the reflector is read once for all four), the four dot products reduced
// together (transposed butterfly: 6 double shuffles instead of 20, then 4 broadcasts)
struct TsApply {
  const double* V;
  int m, n, nb;
  const double* tau;
  const double* Xin;
  int ldin, kq;
  double* Xout;
  int ldout;
};
__global__ void __launch_bounds__(QRR_THREADS) k_tsqr_apply4(const TsApply a0, const TsApply a1) {
  pdl_wait();  // PDL launches: inputs come from the previous TSQR level
  pdl_trigger();
  const TsApply& A = blockIdx.y == 0 ? a0 : a1;  // matrix blockIdx.y (F, G)
  const double* V = A.V;
  const int m = A.m, n = A.n, nb = A.nb, ldin = A.ldin, kq = A.kq, ldout = A.ldout;
  const double *tau = A.tau, *Xin = A.Xin;
  double* Xout = A.Xout;
  extern __shared__ double tv[];  // reflectors rows x n (unit diagonal, zeros above) | tau[n]
  constexpr int PL = TS_ROWS / 32;
  const int i = blockIdx.x, r0 = ts_row0(i, m, nb), rows = ts_row0(i + 1, m, nb) - r0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* tt = tv + size_t(rows) * n;
  for (int e = tid; e < rows * n; e += blockDim.x) {
    const int c = e / rows, r = e - c * rows;
    tv[e] = r > c ? V[size_t(c) * m + r0 + r] : (r == c ? 1.0 : 0.0);
  }
  for (int c = tid; c < n; c += blockDim.x) tt[c] = tau[size_t(i) * n + c];
  __syncthreads();
  for (int q0 = 4 * warp; q0 < kq; q0 += 4 * QRR_WARPS) {
    double y[4][PL];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int u = 0; u < PL; ++u) {
        const int r = lane + 32 * u;
        y[c][u] = (r < n && q0 + c < kq) ? Xin[size_t(q0 + c) * ldin + size_t(i) * n + r] : 0.0;
      }
    const bool b4 = lane & 16, b3 = lane & 8;
    for (int j = n - 1; j >= 0; --j) {
      const double* vj = tv + size_t(j) * rows;
      double vr[PL];
#pragma unroll
      for (int u = 0; u < PL; ++u) {
        const int r = lane + 32 * u;
        vr[u] = (r < rows && r >= j) ? vj[r] : 0.0;
      }
      double s[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int u = 0; u < PL; ++u) acc = fma(vr[u], y[c][u], acc);
        s[c] = acc;
      }
      // xor 16: keep columns {0,1} (bit 4 clear) or {2,3}
      const double k0 = b4 ? s[2] : s[0], k1 = b4 ? s[3] : s[1];
      const double g0 = b4 ? s[0] : s[2], g1 = b4 ? s[1] : s[3];
      const double t0 = k0 + __shfl_xor_sync(0xffffffffu, g0, 16);
      const double t1 = k1 + __shfl_xor_sync(0xffffffffu, g1, 16);
      // xor 8: keep column 2 b4 + b3
      const double kk = b3 ? t1 : t0, gg = b3 ? t0 : t1;
      double t = kk + __shfl_xor_sync(0xffffffffu, gg, 8);
      t += __shfl_xor_sync(0xffffffffu, t, 4);
      t += __shfl_xor_sync(0xffffffffu, t, 2);
      t += __shfl_xor_sync(0xffffffffu, t, 1);
      const double tj = tt[j];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double tw = tj * __shfl_sync(0xffffffffu, t, 8 * c);
#pragma unroll
        for (int u = 0; u < PL; ++u) y[c][u] = fma(-tw, vr[u], y[c][u]);
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int u = 0; u < PL; ++u) {
        const int r = lane + 32 * u;
        if (r < rows && q0 + c < kq) Xout[size_t(q0 + c) * ldout + r0 + r] = y[c][u];
      }
  }
}

// thin Q (compact WY: dlarft / dorg2r order) and the un-pivoted R of a factor left in A by the
// pivoted QR kernels (R above + beta on the diagonal, scaled reflectors below, tau, perm)
void qr_form(ProcWork& w, const double* A, int m, int n, int keep, const double* tau, const int* perm,
             DeviceBuffer& Qb, DeviceBuffer& Rb) {
  ptb_context* ctx = w.ctx;
  cudaStream_t st = ctx->stream;
  double* Q = static_cast<double*>(Qb.get(std::max<size_t>(1, size_t(m) * keep) * sizeof(double)));
  double* R = static_cast<double*>(Rb.get(std::max<size_t>(1, size_t(keep) * n) * sizeof(double)));
  if (keep == 0) return;
  const size_t mk = size_t(m) * keep, kk = size_t(keep) * keep;
  double* V = static_cast<double*>(w.buf[19].get(mk * sizeof(double)));
  double* S = static_cast<double*>(w.buf[20].get(3 * kk * sizeof(double)));
  double* T = S + kk;
  double* W = T + kk;
  k_wy_prep<<<unsigned(std::min<size_t>((mk + 255) / 256, size_t(ctx->num_sms) * 16)), 256, 0, st>>>(A, m, keep, V,
                                                                                                    Q);
  PTB_LAUNCH_CHECK(ctx);
  gemm(ctx, true, false, keep, keep, m, 1.0, V, m, V, m, 0.0, S, keep);  // S = V^T V
  wy_larft(ctx, st, S, tau, keep, T);
  gemm(ctx, false, true, keep, keep, keep, 1.0, T, keep, V, m, 0.0, W, keep);  // W = T V1^T
  gemm(ctx, false, false, m, keep, keep, -1.0, V, m, W, keep, 1.0, Q, m);     // Q = E - V W
  k_unpivot_r<<<std::max(1, std::min(256, (keep * n + 255) / 256)), 256, 0, st>>>(A, m, n, keep, perm, R);
  PTB_LAUNCH_CHECK(ctx);
}

// truncated_qr (procrustes.cpp:34-46): Q (m x keep) and R (keep x n, un-pivoted) in
// caller buffers; A is copied (the input is not modified).  Returns keep.
int truncated_qr_direct(ProcWork& w, const double* A_in, int m, int n, double drop_tol, DeviceBuffer& Qb,
                        DeviceBuffer& Rb) {
  ptb_context* ctx = w.ctx;
  cudaStream_t st = ctx->stream;
  const int k = std::min(m, n);
  if (k == 0) {
    Qb.get(8);
    Rb.get(8);
    return 0;
  }
  double* A = static_cast<double*>(w.buf[0].get(size_t(m) * n * sizeof(double)));
  PTB_CUDA_CHECK(cudaMemcpyAsync(A, A_in, size_t(m) * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  double* tau = static_cast<double*>(w.buf[1].get(size_t(n) * sizeof(double)));
  int* perm = static_cast<int*>(w.buf[2].get(size_t(n) * sizeof(int)));
  int* keep_d = static_cast<int*>(w.buf[3].get(sizeof(int)));
  double* betas = static_cast<double*>(w.buf[5].get(size_t(n) * sizeof(double)));
  const size_t small_smem = (size_t(m) * n + 2 * size_t(n) + 32) * sizeof(double);
  static const bool small_env = [] {  // PTB_QR_SMALL=0 keeps small matrices on the cooperative kernel
    const char* e = std::getenv("PTB_QR_SMALL");
    return !(e && std::atoi(e) == 0);
  }();
  const int reg = !small_env ? 0 : (m <= 128 && n <= 64) ? 1 : (m <= 256 && n <= 64) ? 2 : (m <= 128 && n <= 128) ? 3 : 0;
  if (reg) {  // register-resident pivoted QR (one CTA, two barriers per column)
    QrRegArgs ra{A, m, m, n, 0, 1, drop_tol, A, nullptr, 0, nullptr, 0, tau, perm, keep_d, betas};
    if (reg == 1) launch_pdl(k_qr_reg<4, 4, true, false>, dim3(1), dim3(QRR_THREADS), 0, st, ra, ra);
    else if (reg == 2) launch_pdl(k_qr_reg<4, 8, true, false>, dim3(1), dim3(QRR_THREADS), 0, st, ra, ra);
    else launch_pdl(k_qr_reg<8, 4, true, false>, dim3(1), dim3(QRR_THREADS), 0, st, ra, ra);
    PTB_LAUNCH_CHECK(ctx);
  } else if (small_env && small_smem <= 200 * 1024) {
    QrArgs qa{A, m, n, m, 1, drop_tol, tau, perm, nullptr, keep_d, betas};
    PTB_CUDA_CHECK(
        cudaFuncSetAttribute(k_qrcp_small<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(small_smem)));
    k_qrcp_small<true><<<1, 1024, small_smem, st>>>(qa);
    PTB_LAUNCH_CHECK(ctx);
  } else if (small_env && m <= 1024 && n <= 4096) {
    QrArgs qa{A, m, n, m, 1, drop_tol, tau, perm, nullptr, keep_d, betas};
    const size_t gsmem = (2 * size_t(n) + 32) * sizeof(double);
    PTB_CUDA_CHECK(cudaFuncSetAttribute(k_qrcp_small<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(gsmem)));
    k_qrcp_small<false><<<1, 1024, gsmem, st>>>(qa);
    PTB_LAUNCH_CHECK(ctx);
  } else {
    size_t smem = (QR_THREADS + 2 * size_t(n)) * sizeof(double);
    // matrices too big for k_qrcp_small but with few rows (the corrector's H at cfg4 is ~270^2):
    // spread the rows thinner, the per-column latency rather than bandwidth is what matters
    const int G = qr_grid(ctx, m, smem + 16384 * sizeof(double), reinterpret_cast<const void*>(k_qrcp),
                          m < 8192 ? 64 : 512);
    const size_t rows_per = (size_t(m) + G - 1) / G;
    if (rows_per > 16384) fail(PTB_UNSUPPORTED, "truncated_qr: too many rows per CTA");
    smem += rows_per * sizeof(double);
    double* part = static_cast<double*>(w.buf[4].get(size_t(2) * G * (n + 1) * sizeof(double)));
    QrArgs qa{A, m, n, m, 1, drop_tol, tau, perm, part, keep_d, betas};
    void* args[] = {&qa};
    PTB_CUDA_CHECK(cudaFuncSetAttribute(k_qrcp, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    PTB_CUDA_CHECK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_qrcp), G, QR_THREADS, args, smem, st));
    PTB_LAUNCH_CHECK(ctx);
  }
  int keep = 0;
  PTB_CUDA_CHECK(cudaMemcpyAsync(&keep, keep_d, sizeof(int), cudaMemcpyDeviceToHost, st));
  PTB_CUDA_CHECK(cudaStreamSynchronize(st));
  qr_form(w, A, m, n, keep, tau, perm, Qb, Rb);
  return keep;
}

constexpr int JC_GS_DEFAULT = 4;  // measured: 108^2 2.22 ms (GS 4) vs 2.32 (8), 2.31 (2), 2.80 (1)
size_t jacobi_cluster_smem(int r, int c) {
  const int pairs = ((c % 2 == 0) ? c : c + 1) / 2;
  const int na = (r + JC_CS - 1) / JC_CS + 1, nv = (c + JC_CS - 1) / JC_CS + 1;
  return (size_t(c) * (na + nv) + 2 * size_t(JC_CS + 1) * 4 * pairs + 4 * size_t(c) + 4) * sizeof(double);
}

// thin SVD of M (p x q): U (p x k), sigma (k, host), V (q x k), k = min(p, q)
// One-sided Jacobi of A (r x c, r >= c, column-major, overwritten): A := U (sorted, unit
// columns), V (c x c), sigma (c, descending) -- the device buffers of JacobiArgs.
void jacobi_core(ProcWork& w, double* A, int r, int c, double* V, double* sg, double* tmp, int* order) {
  ptb_context* ctx = w.ctx;
  cudaStream_t st = ctx->stream;
  JacobiArgs ja{A, V, r, c, sg, order, tmp, 40};
  PTB_CUDA_CHECK(cudaMemsetAsync(tmp + size_t(r) * c + size_t(c) * c + c + 17, 0, 5 * sizeof(double), st));
  const size_t smem = (size_t(r) * c + size_t(c) * c) * sizeof(double);
  static const int jacobi_env = [] {  // PTB_JACOBI=single: one-CTA global-memory kernel; =coop: grid
    const char* e = std::getenv("PTB_JACOBI");
    if (e && std::string(e) == "single") return 1;
    if (e && std::string(e) == "coop") return 2;
    if (e && std::string(e) == "small") return 3;  // one-CTA shared-memory kernels only
    return 0;
  }();
  const int pairs = ((c % 2 == 0) ? c : c + 1) / 2;
  const size_t csmem = jacobi_cluster_smem(r, c);
  // measured (scripts/ubench_procrustes.py): the cluster kernel wins from ~64 columns (108: 2.2 vs 3.1 ms),
  // the one-CTA kernel below (60: 0.65 vs 0.72 ms)
  static const int cluster_min = [] {  // PTB_JACOBI_CLUSTER_MIN: smallest c for the cluster kernel
    const char* e = std::getenv("PTB_JACOBI_CLUSTER_MIN");
    return e ? std::atoi(e) : 64;  // measured crossover: 60^2 equal, 80^2 1.30 vs 1.50 ms, 95^2 1.80 vs 2.35 ms
  }();
  const bool cluster_ok = jacobi_env == 0 && c >= cluster_min && pairs * 8 <= 1024 && csmem <= 200 * 1024;
  if (cluster_ok || (smem <= 200 * 1024 && jacobi_env != 2)) {
    if (cluster_ok) {
      static const int gs_env = [] {  // PTB_JACOBI_GS: lanes per pair in the cluster kernel (1, 2, 4, 8)
        const char* e = std::getenv("PTB_JACOBI_GS");
        const int v = e ? std::atoi(e) : 0;
        return (v == 1 || v == 2 || v == 4 || v == 8) ? v : 0;
      }();
      const int gs = gs_env ? gs_env : JC_GS_DEFAULT;
      const void* kern = gs == 1   ? reinterpret_cast<const void*>(k_jacobi_cluster<1>)
                         : gs == 2 ? reinterpret_cast<const void*>(k_jacobi_cluster<2>)
                         : gs == 4 ? reinterpret_cast<const void*>(k_jacobi_cluster<4>)
                                   : reinterpret_cast<const void*>(k_jacobi_cluster<8>);
      PTB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(csmem)));
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(JC_CS);
      cfg.blockDim = dim3(unsigned(std::max(32, (pairs * gs + 31) / 32 * 32)));
      cfg.dynamicSmemBytes = csmem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = JC_CS;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      void* args[] = {&ja};
      PTB_CUDA_CHECK(cudaLaunchKernelExC(&cfg, kern, args));
    } else if (r <= 128 && pairs * 8 <= 512) {  // one 8-lane group per pair, <= 16 rows per lane
      PTB_CUDA_CHECK(
          cudaFuncSetAttribute(k_jacobi_small<8, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      k_jacobi_small<8, 16><<<1, std::max(32, (pairs * 8 + 31) / 32 * 32), smem, st>>>(ja);
    } else if (r <= 256 && pairs * 16 <= 512) {
      PTB_CUDA_CHECK(
          cudaFuncSetAttribute(k_jacobi_small<16, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      k_jacobi_small<16, 16><<<1, std::max(32, (pairs * 16 + 31) / 32 * 32), smem, st>>>(ja);
    } else {
      PTB_CUDA_CHECK(cudaFuncSetAttribute(k_jacobi<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      k_jacobi<true><<<1, 1024, smem, st>>>(ja);
    }
    PTB_LAUNCH_CHECK(ctx);
  } else if (jacobi_env == 1) {
    k_jacobi<false><<<1, 1024, 0, st>>>(ja);
    PTB_LAUNCH_CHECK(ctx);
  } else {
    unsigned long long* ctl = static_cast<unsigned long long*>(w.buf[21].get(8 * sizeof(unsigned long long)));
    const int pairs = ((c % 2 == 0) ? c : c + 1) / 2;
    int per_sm = 0;
    PTB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jacobi_coop, 256, 0));
    const int G = std::max(1, std::min({(pairs + 7) / 8, ctx->num_sms * std::max(1, per_sm), ctx->num_sms}));
    void* args[] = {&ja, &ctl};
    PTB_CUDA_CHECK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_jacobi_coop), G, 256, args, 0, st));
    PTB_LAUNCH_CHECK(ctx);
    k_jacobi_finish<<<1, 1024, 0, st>>>(ja, ctl);
    PTB_LAUNCH_CHECK(ctx);
  }
  if (HostProf(st).on) {  // diagnostics: sweeps used (written after the singular values)
    double d[22] = {};
    PTB_CUDA_CHECK(cudaMemcpyAsync(d, tmp + size_t(r) * c + size_t(c) * c + c, sizeof(d), cudaMemcpyDeviceToHost, st));
    if (d[21] > 0)
      std::fprintf(stderr, "[ptb prof] jacobi cluster cycles/round: partials+send %.0f, wait %.0f, decide+rotate %.0f, barrier %.0f\n",
                   d[17] / d[21], d[18] / d[21], d[19] / d[21], d[20] / d[21]);
    PTB_CUDA_CHECK(cudaStreamSynchronize(st));
    std::fprintf(stderr, "[ptb prof] jacobi %d x %d: %g sweeps; rotations per sweep (cluster kernel):", r, c, d[0]);
    for (int k = 1; k < 17 && k <= int(d[0]) + 1; ++k) std::fprintf(stderr, " %g", d[k]);
    std::fprintf(stderr, "\n");
  }
}

// Tall blocked variant of truncated_qr (m >= 8n): (1) unpivoted Householder QR A = Q1 R1 in
// panels of QB columns -- each panel factored by k_qrcp without pivoting on L2-resident data,
// the trailing matrix updated with compact WY (three DGEMMs); (2) the pivoted QR of the small
// R1 (n x n) by truncated_qr_direct: R1 P = Q2 R2 with the reference's keep rule -- column norms
// are invariant under Q1, so the pivot order and |R_jj| are those of A's own column-pivoted QR
// (procrustes.cpp:37) up to rounding; (3) Q = Q1 [Q2; 0], applying the panels in reverse.
constexpr int QB = 32;

int truncated_qr_blocked(ProcWork& w, const double* A_in, int m, int n, double drop_tol, DeviceBuffer& Qb,
                         DeviceBuffer& Rb) {
  ptb_context* ctx = w.ctx;
  cudaStream_t st = ctx->stream;
  double* A = static_cast<double*>(w.BA.get(size_t(m) * n * sizeof(double)));
  double* V = static_cast<double*>(w.BV.get(size_t(m) * n * sizeof(double)));
  PTB_CUDA_CHECK(cudaMemcpyAsync(A, A_in, size_t(m) * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  const int P = (n + QB - 1) / QB;
  double* tau = static_cast<double*>(w.BT.get((size_t(n) + size_t(P) * QB * QB + 3 * size_t(QB) * n) *
                                              sizeof(double)));
  double* Tall = tau + n;               // P x (QB x QB)
  double* W1 = Tall + size_t(P) * QB * QB;  // QB x n
  double* W2 = W1 + size_t(QB) * n;         // QB x n
  double* S = W2 + size_t(QB) * n;          // QB x QB (<= QB x n)
  int* perm = static_cast<int*>(w.buf[2].get(size_t(n) * sizeof(int)));
  int* keep_d = static_cast<int*>(w.buf[3].get(sizeof(int)));
  double* betas = static_cast<double*>(w.buf[5].get(size_t(n) * sizeof(double)));
  for (int p = 0; p < P; ++p) {
    const int c0 = p * QB, wd = std::min(QB, n - c0), mp = m - c0, nr = n - c0 - wd;
    double* Ap = A + size_t(c0) * m + c0;
    const size_t smem0 = (size_t(wd) + QR_THREADS) * sizeof(double);
    const int G = qr_grid(ctx, mp, smem0 + 2 * 8192 * sizeof(double), reinterpret_cast<const void*>(k_qr_panel));
    const size_t rows_per = (size_t(mp) + G - 1) / G;
    if (rows_per > 8192) fail(PTB_UNSUPPORTED, "truncated_qr: too many rows per CTA");
    const size_t smem = smem0 + 2 * rows_per * sizeof(double);
    double* part = static_cast<double*>(w.buf[4].get(size_t(2) * G * (wd + 1) * sizeof(double)));
    double* rowb = static_cast<double*>(w.buf[22].get(size_t(2) * wd * sizeof(double)));
    PanelArgs pa{Ap, mp, wd, m, tau + c0, part, rowb};
    void* args[] = {&pa};
    PTB_CUDA_CHECK(cudaFuncSetAttribute(k_qr_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    PTB_CUDA_CHECK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_qr_panel), G, QR_THREADS, args, smem, st));
    PTB_LAUNCH_CHECK(ctx);
    double* Vp = V + size_t(c0) * m + c0;
    k_panel_v<<<unsigned(std::min<size_t>((size_t(mp) * wd + 255) / 256, size_t(ctx->num_sms) * 16)), 256, 0, st>>>(
        Ap, m, mp, wd, Vp);
    PTB_LAUNCH_CHECK(ctx);
    double* Tp = Tall + size_t(p) * QB * QB;
    gemm(ctx, true, false, wd, wd, mp, 1.0, Vp, m, Vp, m, 0.0, S, wd);  // S = Vp^T Vp
    wy_larft(ctx, st, S, tau + c0, wd, Tp);
    if (nr > 0) {  // A_trail -= Vp (Tp^T (Vp^T A_trail))
      double* At = A + size_t(c0 + wd) * m + c0;
      gemm(ctx, true, false, wd, nr, mp, 1.0, Vp, m, At, m, 0.0, W1, wd);
      gemm(ctx, true, false, wd, nr, wd, 1.0, Tp, wd, W1, wd, 0.0, W2, wd);
      gemm(ctx, false, false, mp, nr, wd, -1.0, Vp, m, W2, wd, 1.0, At, m);
    }
  }
  // R1 and its pivoted QR
  double* R1 = static_cast<double*>(w.BR.get(size_t(n) * n * sizeof(double)));
  k_triu<<<unsigned(std::max(1, std::min(1024, (n * n + 255) / 256))), 256, 0, st>>>(A, m, n, R1);
  PTB_LAUNCH_CHECK(ctx);
  const int kq = truncated_qr_direct(w, R1, n, n, drop_tol, w.BQ2, Rb);
  double* Q = static_cast<double*>(Qb.get(std::max<size_t>(1, size_t(m) * kq) * sizeof(double)));
  if (kq == 0) return 0;
  // Q = Q1 [Q2; 0]
  PTB_CUDA_CHECK(cudaMemsetAsync(Q, 0, size_t(m) * kq * sizeof(double), st));
  PTB_CUDA_CHECK(cudaMemcpy2DAsync(Q, size_t(m) * sizeof(double), w.BQ2.ptr, size_t(n) * sizeof(double),
                                   size_t(n) * sizeof(double), kq, cudaMemcpyDeviceToDevice, st));
  double* Y1 = W1;  // QB x kq (kq <= n)
  double* Y2 = W2;
  for (int p = P - 1; p >= 0; --p) {
    const int c0 = p * QB, wd = std::min(QB, n - c0), mp = m - c0;
    const double* Vp = V + size_t(c0) * m + c0;
    const double* Tp = Tall + size_t(p) * QB * QB;
    double* Xp = Q + c0;  // rows c0.., ld m
    gemm(ctx, true, false, wd, kq, mp, 1.0, Vp, m, Xp, m, 0.0, Y1, wd);
    gemm(ctx, false, false, wd, kq, wd, 1.0, Tp, wd, Y1, wd, 0.0, Y2, wd);
    gemm(ctx, false, false, mp, kq, wd, -1.0, Vp, m, Y2, wd, 1.0, Xp, m);
  }
  return kq;
}

// TSQR route of truncated_qr (see the TSQR note above k_qr_reg): up-sweep of leaf QRs, the pivoted QR of the
// last stack with the reference's keep rule, then the down-sweep forming Q = Q_0 ... Q_L Q_top.
int truncated_qr_tsqr(ProcWork& w, const double* A_in, int m, int n, double drop_tol, DeviceBuffer& Qb,
                      DeviceBuffer& Rb) {
  ptb_context* ctx = w.ctx;
  cudaStream_t st = ctx->stream;
  struct Level {
    int m, nb;
    double *V, *tau;
  };
  std::vector<Level> lv;
  const double* cur = A_in;
  int curm = m, ld = m;
  PTB_CUDA_CHECK(cudaFuncSetAttribute(k_tsqr_apply4, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int((size_t(TS_ROWS) * TS_MAXN + TS_MAXN) * sizeof(double))));
  while (curm > TS_ROWS) {
    const int L = int(lv.size());
    if (3 * L + 2 >= int(sizeof(w.TS) / sizeof(w.TS[0]))) fail(PTB_UNSUPPORTED, "truncated_qr: TSQR depth");
    const int nb = (curm + TS_ROWS - 1) / TS_ROWS;
    const int rows_max = (curm + nb - 1) / nb;
    double* V = static_cast<double*>(w.TS[3 * L].get(size_t(curm) * n * sizeof(double)));
    double* tau = static_cast<double*>(w.TS[3 * L + 1].get(size_t(nb) * n * sizeof(double)));
    double* S = static_cast<double*>(w.TS[3 * L + 2].get(size_t(nb) * n * n * sizeof(double)));
    (void)rows_max;
    QrRegArgs la{cur, ld, curm, n, nb, 0, -1.0, nullptr, V, curm, S, nb * n, tau, nullptr, nullptr, nullptr};
    launch_pdl(k_qr_reg<4, 8, false, true>, dim3(unsigned(nb)), dim3(QRR_THREADS), 0, st, la, la);
    PTB_LAUNCH_CHECK(ctx);
    lv.push_back(Level{curm, nb, V, tau});
    cur = S;
    curm = nb * n;
    ld = curm;
  }
  const int kq = truncated_qr_direct(w, cur, curm, n, drop_tol, w.BQ2, Rb);
  double* Q = static_cast<double*>(Qb.get(std::max<size_t>(1, size_t(m) * kq) * sizeof(double)));
  if (kq == 0) return 0;
  const double* X = static_cast<const double*>(w.BQ2.ptr);
  int ldx = curm;
  for (int l = int(lv.size()) - 1; l >= 0; --l) {
    const Level& L = lv[size_t(l)];
    double* out = l == 0 ? Q : static_cast<double*>(w.TX[l & 1].get(size_t(L.m) * kq * sizeof(double)));
    const int rows_max = (L.m + L.nb - 1) / L.nb;
    const TsApply ap{L.V, L.m, n, L.nb, L.tau, X, ldx, kq, out, L.m};
    launch_pdl(k_tsqr_apply4, dim3(unsigned(L.nb)), dim3(QRR_THREADS), (size_t(rows_max) * n + n) * sizeof(double), st, ap, ap);
    PTB_LAUNCH_CHECK(ctx);
    X = out;
    ldx = L.m;
  }
  if (lv.empty())
    PTB_CUDA_CHECK(cudaMemcpyAsync(Q, X, size_t(m) * kq * sizeof(double), cudaMemcpyDeviceToDevice, st));
  return kq;
}

// R (k1 + k2) x (n1 + n2), column-major: [R1 C; 0 R2] with C = C1 + C2 (the two Gram-Schmidt passes)
__global__ void k_assemble_r2(int k1, int k2, int n1, int n2, const double* R1, const double* C1, const double* C2,
                              const double* R2, double* R) {
  const int rows = k1 + k2, cols = n1 + n2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += gridDim.x * blockDim.x) {
    const int j = e / rows, i = e - j * rows;
    double x = 0.0;
    if (j < n1) {
      if (i < k1) x = R1[size_t(j) * k1 + i];
    } else if (i < k1) {
      x = C1[size_t(j - n1) * k1 + i] + C2[size_t(j - n1) * k1 + i];
    } else {
      x = R2[size_t(j - n1) * k2 + (i - k1)];
    }
    R[e] = x;
  }
}

// Tall blocks of TS_MAXN < n <= 2 TS_MAXN columns (config 4's update_svd: 196608 x 128): the first
// 64 columns through the TSQR route, the rest projected off its Q by block Gram-Schmidt applied
// twice (BCGS2: orthogonal to working precision), their TSQR, then the column-pivoted QR of the
// assembled R = [R1 C; 0 R2].  A = [Q1 Q2] R with [Q1 Q2] orthonormal, so the pivoting and keep
// decisions are those of A's own column-pivoted QR (procrustes.cpp:34-46) up to rounding, as for
// the TSQR route; Q = [Q1 Q2] Q_R.  Replaces the blocked route (one grid barrier per column).
int truncated_qr_2panel(ProcWork& w, const double* A_in, int m, int n, double drop_tol, DeviceBuffer& Qb,
                        DeviceBuffer& Rb) {
  ptb_context* ctx = w.ctx;
  cudaStream_t st = ctx->stream;
  const int n1 = TS_MAXN, n2 = n - n1;
  const int k1 = truncated_qr_tsqr(w, A_in, m, n1, 0.0, w.TP[0], w.TP[1]);
  const double* Q1 = static_cast<const double*>(w.TP[0].ptr);
  double* A2 = static_cast<double*>(w.TP[2].get(size_t(m) * n2 * sizeof(double)));
  PTB_CUDA_CHECK(cudaMemcpyAsync(A2, A_in + size_t(n1) * m, size_t(m) * n2 * sizeof(double), cudaMemcpyDeviceToDevice,
                                 st));
  double* C = static_cast<double*>(w.TP[3].get(std::max<size_t>(1, 2 * size_t(k1) * n2) * sizeof(double)));
  if (k1 > 0) {
    for (int pass = 0; pass < 2; ++pass) {
      double* Cp = C + size_t(pass) * k1 * n2;
      gemm(ctx, true, false, k1, n2, m, 1.0, Q1, m, A2, m, 0.0, Cp, k1);
      gemm(ctx, false, false, m, n2, k1, -1.0, Q1, m, Cp, k1, 1.0, A2, m);
    }
  }
  const int k2 = truncated_qr_tsqr(w, A2, m, n2, 0.0, w.TP[4], w.TP[5]);
  const int kk = k1 + k2;
  double* R = static_cast<double*>(w.TP[6].get(std::max<size_t>(1, size_t(kk) * n) * sizeof(double)));
  if (kk == 0) {
    Qb.get(8);
    Rb.get(8);
    return 0;
  }
  k_assemble_r2<<<unsigned(std::max(1, std::min(1024, (kk * n + 255) / 256))), 256, 0, st>>>(
      k1, k2, n1, n2, static_cast<const double*>(w.TP[1].ptr), C, C + size_t(k1) * n2,
      static_cast<const double*>(w.TP[5].ptr), R);
  PTB_LAUNCH_CHECK(ctx);
  const int kq = truncated_qr_direct(w, R, kk, n, drop_tol, w.BQ2, Rb);
  double* Q = static_cast<double*>(Qb.get(std::max<size_t>(1, size_t(m) * kq) * sizeof(double)));
  if (kq == 0) return 0;
  const double* QR = static_cast<const double*>(w.BQ2.ptr);  // kk x kq
  if (k1 > 0) gemm(ctx, false, false, m, kq, k1, 1.0, Q1, m, QR, kk, 0.0, Q, m);
  if (k2 > 0)
    gemm(ctx, false, false, m, kq, k2, 1.0, static_cast<const double*>(w.TP[4].ptr), m, QR + k1, kk,
         k1 > 0 ? 1.0 : 0.0, Q, m);
  return kq;
}

// PTB_QR=direct | blocked | tsqr forces a route (tests, diagnostics); 0 = automatic
int qr_route_env() {
  static const int env = [] {
    const char* e = std::getenv("PTB_QR");
    if (!e) return 0;
    const std::string v(e);
    return v == "direct" ? 1 : v == "blocked" ? 2 : v == "tsqr" ? 3 : v == "panel2" ? 4 : 0;
  }();
  return env;
}

// update_svd's two QRs (F and G: same shape) through the TSQR route together: every leaf level
// and every down-sweep level is one launch for both matrices, the two pivoted QRs of the last
// stacks are one launch, and one host synchronisation reads both keep counts.  Each matrix goes
// through exactly the arithmetic of truncated_qr_tsqr.  Returns false (nothing done) when the
// shape is not a TSQR shape.
bool truncated_qr_pair(ProcWork& w, const double* F, const double* G, int m, int n, double tol_f, double tol_g,
                       DeviceBuffer& QF, DeviceBuffer& RF, DeviceBuffer& QG, DeviceBuffer& RG, int& kf, int& kg) {
  if (!(m >= 8 * n && m > 1024 && n <= TS_MAXN && n > 0) || qr_route_env() != 0) return false;
  ptb_context* ctx = w.ctx;
  cudaStream_t st = ctx->stream;
  struct Level {
    int m, nb;
    double *V[2], *tau[2];
  };
  std::vector<Level> lv;
  const double* cur[2] = {F, G};
  int curm = m, ld = m;
  PTB_CUDA_CHECK(cudaFuncSetAttribute(k_tsqr_apply4, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int((size_t(TS_ROWS) * TS_MAXN + TS_MAXN) * sizeof(double))));
  while (curm > TS_ROWS) {
    const int L = int(lv.size());
    if (3 * L + 2 >= int(sizeof(w.TS) / sizeof(w.TS[0]))) fail(PTB_UNSUPPORTED, "truncated_qr: TSQR depth");
    const int nb = (curm + TS_ROWS - 1) / TS_ROWS;
    Level lev{curm, nb, {}, {}};
    QrRegArgs la[2];
    double* S[2];
    for (int b = 0; b < 2; ++b) {
      DeviceBuffer* T = b == 0 ? w.TS : w.TS2;
      lev.V[b] = static_cast<double*>(T[3 * L].get(size_t(curm) * n * sizeof(double)));
      lev.tau[b] = static_cast<double*>(T[3 * L + 1].get(size_t(nb) * n * sizeof(double)));
      S[b] = static_cast<double*>(T[3 * L + 2].get(size_t(nb) * n * n * sizeof(double)));
      la[b] = QrRegArgs{cur[b], ld, curm, n, nb, 0, -1.0, nullptr, lev.V[b], curm, S[b], nb * n, lev.tau[b],
                        nullptr, nullptr, nullptr};
    }
    launch_pdl(k_qr_reg<4, 8, false, true>, dim3(unsigned(nb), 2), dim3(QRR_THREADS), 0, st, la[0], la[1]);
    PTB_LAUNCH_CHECK(ctx);
    lv.push_back(lev);
    cur[0] = S[0];
    cur[1] = S[1];
    curm = nb * n;
    ld = curm;
  }
  // pivoted QRs of the two last stacks (curm <= TS_ROWS rows), one launch, one sync
  double* A[2];
  double* tau[2];
  int* perm[2];
  int* keep_d = static_cast<int*>(w.buf[3].get(2 * sizeof(int)));
  QrRegArgs ra[2];
  const double tol[2] = {tol_f, tol_g};
  for (int b = 0; b < 2; ++b) {
    DeviceBuffer* P = b == 0 ? w.PA : w.PB;  // [0] factor, [1] tau, [2] perm, [3] |R_jj|
    A[b] = static_cast<double*>(P[0].get(size_t(curm) * n * sizeof(double)));
    tau[b] = static_cast<double*>(P[1].get(size_t(n) * sizeof(double)));
    perm[b] = static_cast<int*>(P[2].get(size_t(n) * sizeof(int)));
    double* betas = static_cast<double*>(P[3].get(size_t(n) * sizeof(double)));
    PTB_CUDA_CHECK(cudaMemcpyAsync(A[b], cur[b], size_t(curm) * n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    ra[b] = QrRegArgs{A[b], curm, curm, n, 0, 1, tol[b], A[b], nullptr, 0, nullptr, 0, tau[b], perm[b], keep_d + b,
                      betas};
  }
  if (curm <= 128) launch_pdl(k_qr_reg<4, 4, true, false>, dim3(2), dim3(QRR_THREADS), 0, st, ra[0], ra[1]);
  else launch_pdl(k_qr_reg<4, 8, true, false>, dim3(2), dim3(QRR_THREADS), 0, st, ra[0], ra[1]);
  PTB_LAUNCH_CHECK(ctx);
  int keep[2] = {0, 0};
  PTB_CUDA_CHECK(cudaMemcpyAsync(keep, keep_d, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  PTB_CUDA_CHECK(cudaStreamSynchronize(st));
  DeviceBuffer* Qt[2] = {&w.BQ2, &w.BQ2b};
  DeviceBuffer* Qo[2] = {&QF, &QG};
  DeviceBuffer* Ro[2] = {&RF, &RG};
  for (int b = 0; b < 2; ++b) {
    qr_form(w, A[b], curm, n, keep[b], tau[b], perm[b], *Qt[b], *Ro[b]);
    Qo[b]->get(std::max<size_t>(1, size_t(m) * keep[b]) * sizeof(double));
  }
  kf = keep[0];
  kg = keep[1];
  if (lv.empty()) {
    for (int b = 0; b < 2; ++b)
      if (keep[b] > 0)
        PTB_CUDA_CHECK(cudaMemcpyAsync(Qo[b]->ptr, Qt[b]->ptr, size_t(m) * keep[b] * sizeof(double),
                                       cudaMemcpyDeviceToDevice, st));
    return true;
  }
  const double* X[2] = {static_cast<const double*>(w.BQ2.ptr), static_cast<const double*>(w.BQ2b.ptr)};
  int ldx = curm;
  for (int l = int(lv.size()) - 1; l >= 0; --l) {
    const Level& L = lv[size_t(l)];
    TsApply ap[2];
    double* out[2];
    for (int b = 0; b < 2; ++b) {
      DeviceBuffer* TX = b == 0 ? w.TX : w.TX2;
      out[b] = l == 0 ? static_cast<double*>(Qo[b]->ptr)
                      : static_cast<double*>(TX[l & 1].get(std::max<size_t>(1, size_t(L.m) * keep[b]) *
                                                           sizeof(double)));
      ap[b] = TsApply{L.V[b], L.m, n, L.nb, L.tau[b], X[b], ldx, keep[b], out[b], L.m};
    }
    const int rows_max = (L.m + L.nb - 1) / L.nb;
    if (keep[0] > 0 || keep[1] > 0) {
      launch_pdl(k_tsqr_apply4, dim3(unsigned(L.nb), 2), dim3(QRR_THREADS), (size_t(rows_max) * n + n) * sizeof(double),
                 st, ap[0], ap[1]);
      PTB_LAUNCH_CHECK(ctx);
    }
    X[0] = out[0];
    X[1] = out[1];
    ldx = L.m;
  }
  return true;
}

int truncated_qr(ProcWork& w, const double* A_in, int m, int n, double drop_tol, DeviceBuffer& Qb, DeviceBuffer& Rb) {
  const int env = qr_route_env();
  const bool tall = m >= 8 * n && m > TS_ROWS;
  if (env == 1) return truncated_qr_direct(w, A_in, m, n, drop_tol, Qb, Rb);
  if (env == 3 && tall && n <= TS_MAXN) return truncated_qr_tsqr(w, A_in, m, n, drop_tol, Qb, Rb);
  if (env == 2 && tall && n > 1) return truncated_qr_blocked(w, A_in, m, n, drop_tol, Qb, Rb);
  if (env == 0 && tall && n <= TS_MAXN && m > 1024) return truncated_qr_tsqr(w, A_in, m, n, drop_tol, Qb, Rb);
  if ((env == 0 || env == 4) && tall && n > TS_MAXN && n <= 2 * TS_MAXN && m > 1024)
    return truncated_qr_2panel(w, A_in, m, n, drop_tol, Qb, Rb);
  if (env == 0 && tall && n > QB) return truncated_qr_blocked(w, A_in, m, n, drop_tol, Qb, Rb);
  return truncated_qr_direct(w, A_in, m, n, drop_tol, Qb, Rb);
}

// thin SVD of M (p x q): U (p x k), sigma (k, host), V (q x k), k = min(p, q).
// A = M (or M^T) is r x c with r >= c.  For c >= 32 it is preconditioned as in dgesvj: a
// column-pivoted QR A = Q R first, then one-sided Jacobi on R^T (c x kq), whose columns are
// already close to orthogonal for graded matrices, so far fewer sweeps are needed (the
// corrector's H spans ~13 decades: 16-24 sweeps unpreconditioned).  R^T = U' S V'^T gives
// A = (Q V') S U'^T.  Row order does not change column inner products, so the un-pivoted R
// truncated_qr returns serves as well as the pivoted one.
void thin_svd(ProcWork& w, const double* M, int p, int q, DeviceBuffer& Ub, std::vector<double>& sigma,
              DeviceBuffer& Vb) {
  ptb_context* ctx = w.ctx;
  cudaStream_t st = ctx->stream;
  const int k = std::min(p, q);
  sigma.assign(size_t(k), 0.0);
  if (k == 0) {
    Ub.get(8);
    Vb.get(8);
    return;
  }
  const bool trans = p < q;
  const int r = trans ? q : p, c = k;
  double* A = static_cast<double*>(w.buf[6].get(size_t(r) * c * sizeof(double)));
  if (trans) {
    k_transpose<<<std::max(1, std::min(1024, (p * q + 255) / 256)), 256, 0, st>>>(M, p, q, A);
    PTB_LAUNCH_CHECK(ctx);
  } else {
    PTB_CUDA_CHECK(cudaMemcpyAsync(A, M, size_t(p) * q * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  static const bool precond_env = [] {
    const char* e = std::getenv("PTB_SVD_PRECOND");
    return !(e && std::atoi(e) == 0);
  }();
  double* U = static_cast<double*>(Ub.get(size_t(p) * k * sizeof(double)));
  double* Vo = static_cast<double*>(Vb.get(size_t(q) * k * sizeof(double)));
  if (precond_env && c >= 32) {
    HostProf hp_(st);
    const int kq = truncated_qr(w, A, r, c, 0.0, w.PQ, w.PR);  // A = Q R, Q r x kq, R kq x c
    hp_.mark("svd: precondition qr");
    double* Bt = static_cast<double*>(w.buf[6].get(size_t(r) * c * sizeof(double)));  // A no longer needed
    double* V = static_cast<double*>(w.buf[7].get(std::max<size_t>(1, size_t(kq) * kq) * sizeof(double)));
    double* sg = static_cast<double*>(w.buf[8].get(size_t(c) * sizeof(double)));
    int* order = static_cast<int*>(w.buf[9].get(size_t(c) * sizeof(int)));
    double* tmp = static_cast<double*>(w.buf[10].get((size_t(r) * c + size_t(c) * c + c + 22) * sizeof(double)));
    std::vector<double> s_k(size_t(kq), 0.0);
    if (kq > 0) {
      // Bt = R^T (c x kq): R is kq x c column-major
      k_transpose<<<std::max(1, std::min(1024, (kq * c + 255) / 256)), 256, 0, st>>>(static_cast<double*>(w.PR.ptr),
                                                                                   kq, c, Bt);
      PTB_LAUNCH_CHECK(ctx);
      jacobi_core(w, Bt, c, kq, V, sg, tmp, order);  // Bt := U' (c x kq), V' (kq x kq)
      hp_.mark("svd: jacobi");
      PTB_CUDA_CHECK(cudaMemcpyAsync(s_k.data(), sg, size_t(kq) * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    // left factor of A: Q V' (r x kq); right factor: U' (c x kq); columns kq..k-1 (sigma 0): zero
    double* QV = static_cast<double*>(w.PU.get(size_t(r) * k * sizeof(double)));
    PTB_CUDA_CHECK(cudaMemsetAsync(QV, 0, size_t(r) * k * sizeof(double), st));
    if (kq > 0) gemm(ctx, false, false, r, kq, kq, 1.0, static_cast<double*>(w.PQ.ptr), r, V, kq, 0.0, QV, r);
    double* UL = trans ? U : Vo;  // destination of U' (c rows)
    double* AL = trans ? Vo : U;  // destination of Q V' (r rows)
    PTB_CUDA_CHECK(cudaMemsetAsync(UL, 0, size_t(c) * k * sizeof(double), st));
    if (kq > 0)
      PTB_CUDA_CHECK(cudaMemcpyAsync(UL, Bt, size_t(c) * kq * sizeof(double), cudaMemcpyDeviceToDevice, st));
    PTB_CUDA_CHECK(cudaMemcpyAsync(AL, QV, size_t(r) * k * sizeof(double), cudaMemcpyDeviceToDevice, st));
    PTB_CUDA_CHECK(cudaStreamSynchronize(st));
    for (int i = 0; i < kq; ++i) sigma[size_t(i)] = s_k[size_t(i)];
    return;
  }
  double* V = static_cast<double*>(w.buf[7].get(size_t(c) * c * sizeof(double)));
  double* sg = static_cast<double*>(w.buf[8].get(size_t(c) * sizeof(double)));
  int* order = static_cast<int*>(w.buf[9].get(size_t(c) * sizeof(int)));
  double* tmp = static_cast<double*>(w.buf[10].get((size_t(r) * c + size_t(c) * c + c + 22) * sizeof(double)));
  jacobi_core(w, A, r, c, V, sg, tmp, order);
  PTB_CUDA_CHECK(cudaMemcpyAsync(sigma.data(), sg, size_t(c) * sizeof(double), cudaMemcpyDeviceToHost, st));
  // M = A_sorted diag(s) V^T  (A is r x c = U when !trans; when trans, M^T = A S V^T -> M = V S A^T)
  if (!trans) {
    PTB_CUDA_CHECK(cudaMemcpyAsync(U, A, size_t(p) * k * sizeof(double), cudaMemcpyDeviceToDevice, st));
    PTB_CUDA_CHECK(cudaMemcpyAsync(Vo, V, size_t(q) * k * sizeof(double), cudaMemcpyDeviceToDevice, st));
  } else {
    PTB_CUDA_CHECK(cudaMemcpyAsync(U, V, size_t(p) * k * sizeof(double), cudaMemcpyDeviceToDevice, st));
    PTB_CUDA_CHECK(cudaMemcpyAsync(Vo, A, size_t(q) * k * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  PTB_CUDA_CHECK(cudaStreamSynchronize(st));
}

static int truncate_count(const std::vector<double>& sigma, double tol) {
  const double smax = sigma.empty() ? 0.0 : sigma[0];
  int keep = 0;
  while (keep < int(sigma.size()) && smax > 0.0 && sigma[size_t(keep)] / smax > tol) ++keep;
  return keep;
}

void fix_signs(ptb_context* ctx, double* X, double* Y, int rows, int cols) {
  if (cols == 0 || rows == 0) return;
  k_fix_signs<<<cols, 256, 0, ctx->stream>>>(X, Y, rows);
  PTB_LAUNCH_CHECK(ctx);
}

void check_tol(double tol) {
  if (!(tol > 0.0) || !(tol < 1.0)) fail(PTB_INVALID_ARGUMENT, "truncation tolerance must lie in (0, 1)");
}

// procrustes.cpp:48-69
void solve_from_scratch(ProcWork& w, DevCorrector& out, const double* F, const double* G, int rows, int cols,
                        double tol) {
  ptb_context* ctx = w.ctx;
  const double qr_guard = 1e-14;
  const double fn = std::sqrt(dev_sumsq(ctx, F, size_t(rows) * cols, w.buf[11]));
  const double gn = std::sqrt(dev_sumsq(ctx, G, size_t(rows) * cols, w.buf[11]));
  const int qf = truncated_qr(w, F, rows, cols, qr_guard * fn, w.QF, w.RF);
  const int qg = truncated_qr(w, G, rows, cols, qr_guard * gn, w.QG, w.RG);
  if (qf == 0 || qg == 0) {
    out.X.get(8);
    out.Y.get(8);
    out.assign(rows, 0, {}, tol);
    return;
  }
  double* M = static_cast<double*>(w.buf[12].get(size_t(qf) * qg * sizeof(double)));
  gemm(ctx, false, true, qf, qg, cols, 1.0, static_cast<double*>(w.RF.ptr), qf, static_cast<double*>(w.RG.ptr), qg,
       0.0, M, qf);
  std::vector<double> sigma;
  thin_svd(w, M, qf, qg, w.Uh, sigma, w.Vh);
  const int s = truncate_count(sigma, tol);
  double* X = static_cast<double*>(out.X.get(std::max<size_t>(1, size_t(rows) * s) * sizeof(double)));
  double* Y = static_cast<double*>(out.Y.get(std::max<size_t>(1, size_t(rows) * s) * sizeof(double)));
  gemm(ctx, false, false, rows, s, qf, 1.0, static_cast<double*>(w.QF.ptr), rows, static_cast<double*>(w.Uh.ptr), qf,
       0.0, X, rows);
  gemm(ctx, false, false, rows, s, qg, 1.0, static_cast<double*>(w.QG.ptr), rows, static_cast<double*>(w.Vh.ptr), qg,
       0.0, Y, rows);
  fix_signs(ctx, X, Y, rows, s);
  sigma.resize(size_t(s));
  out.assign(rows, s, sigma, tol);
}

// procrustes.cpp:188-237; `c` is updated in place.
// ---- row-sharded update_svd -------------------------------------------------------------------
// The corrector's tall matrices (3 N_c rows) are cut into SLABS fixed slabs of whole TSQR leaves;
// with W ranks, rank q owns the contiguous slabs [q SLABS/W, (q+1) SLABS/W).  The products over rows
// (U^T F, V^T G, the panels' Gram-Schmidt projections) are per-slab partials gathered and summed in
// slab order; row-local products (projections, rotations) are never split over k; the TSQR leaves
// of a slab are factored by its owner and the stack of all leaves' R is gathered and reduced by
// every rank (truncated_qr_tsqr on the stack: exactly the unsharded TSQR's levels above the
// leaves).  So every value is the same at any W, W = 1 included; the new factors' own rows are
// gathered, fix_signs and everything small (H, its SVD) are replicated.
constexpr int SLABS = 48;
struct RowPart {
  int W, rank, rows, own, r0;  // own rows [r0, r0 + own)
};

bool row_shard(int rows, int cols, const Comm* comm, RowPart& rp) {
  const int W = comm ? comm->world : 1;
  static const bool env = [] {
    const char* e = std::getenv("PTB_ROW_SHARD");
    return !(e && std::atoi(e) == 0);
  }();
  if (!env || rows % (SLABS * TS_ROWS) != 0 || SLABS % W != 0 || cols < 1 || cols > 2 * TS_MAXN || rows < 8 * cols)
    return false;
  const int rank = comm ? comm->rank : 0;
  rp = RowPart{W, rank, rows, rows / W, rank * (rows / W)};
  return true;
}

// full[(q own + i) + j rows] = g[q own cols + i + j own]: the ranks' row blocks into one matrix
__global__ void k_repack_rows(int W, int own, int cols, const double* __restrict__ g, double* __restrict__ full) {
  const size_t rows = size_t(W) * own, total = rows * size_t(cols);
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t j = e / rows, i = e - j * rows, q = i / size_t(own), li = i - q * size_t(own);
    full[e] = g[q * size_t(own) * cols + li + j * size_t(own)];
  }
}

// every rank's own block (own x cols, ld own) -> full (rows x cols, ld rows) on every rank
void gather_rows(ProcWork& w, const RowPart& rp, const double* own, int cols, double* full, DeviceBuffer& tmp) {
  ptb_context* ctx = w.ctx;
  cudaStream_t st = ctx->stream;
  if (cols == 0) return;
  if (rp.W == 1) {
    if (own != full)
      PTB_CUDA_CHECK(cudaMemcpyAsync(full, own, size_t(rp.rows) * cols * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return;
  }
  double* g = static_cast<double*>(tmp.get(size_t(rp.rows) * cols * sizeof(double)));
  w.comm->allgather(own, g, size_t(rp.own) * cols * sizeof(double), st);
  const size_t total = size_t(rp.rows) * cols;
  k_repack_rows<<<unsigned(std::min<size_t>((total + 255) / 256, size_t(ctx->num_sms) * 8)), 256, 0, st>>>(
      rp.W, rp.own, cols, g, full);
  PTB_LAUNCH_CHECK(ctx);
}

// C (m x n) = A^T B over the slabs: A, B full (every rank holds all rows: z offset = own slabs) or
// own (rows from the own slabs' first row: offset 0)
void slab_tn(ProcWork& w, const RowPart& rp, bool full, int m, int n, const double* A, int lda, const double* B, int ldb,
             double* C) {
  ptb_context* ctx = w.ctx;
  if (m == 0 || n == 0) return;
  const int per = SLABS / rp.W, slab = rp.rows / SLABS;
  double* own = static_cast<double*>(w.SH[6].get(size_t(per) * m * n * sizeof(double)));
  double* all = rp.W == 1 ? own : static_cast<double*>(w.SH[7].get(size_t(SLABS) * m * n * sizeof(double)));
  gemm_tn_slabs(ctx, m, n, A, lda, B, ldb, C, m, SLABS, slab, full ? rp.rank * per : 0, per, own, all, [&] {
    if (rp.W > 1) w.comm->allgather(own, all, size_t(per) * m * n * sizeof(double), ctx->stream);
  });
}

// truncated_qr (procrustes.cpp:34-46) of a row-sharded tall block through the TSQR route: this
// rank's leaves, the gathered stack of all leaves' R reduced by truncated_qr_tsqr (the unsharded
// TSQR above its first level), then this rank's leaves applied to the stack's Q -> the own rows of
// Q (own x kq, ld own).  R and kq are the same on every rank.
int tsqr_rows(ProcWork& w, const RowPart& rp, const double* A, int lda, int n, double drop_tol, DeviceBuffer& Qo,
              DeviceBuffer& Rb) {
  ptb_context* ctx = w.ctx;
  cudaStream_t st = ctx->stream;
  const int nbo = rp.own / TS_ROWS, nbt = rp.rows / TS_ROWS;
  double* V = static_cast<double*>(w.SH[0].get(size_t(rp.own) * n * sizeof(double)));
  double* tau = static_cast<double*>(w.SH[1].get(size_t(nbo) * n * sizeof(double)));
  double* So = static_cast<double*>(w.SH[2].get(size_t(nbo) * n * n * sizeof(double)));
  QrRegArgs la{A, lda, rp.own, n, nbo, 0, -1.0, nullptr, V, rp.own, So, nbo * n, tau, nullptr, nullptr, nullptr};
  launch_pdl(k_qr_reg<4, 8, false, true>, dim3(unsigned(nbo)), dim3(QRR_THREADS), 0, st, la, la);
  PTB_LAUNCH_CHECK(ctx);
  double* S = So;
  if (rp.W > 1) {
    S = static_cast<double*>(w.SH[3].get(size_t(nbt) * n * n * sizeof(double)));
    RowPart sp{rp.W, rp.rank, nbt * n, nbo * n, rp.rank * nbo * n};  // the stack: rows = leaves x n
    gather_rows(w, sp, So, n, S, w.SH[4]);
  }
  const int kq = truncated_qr_tsqr(w, S, nbt * n, n, drop_tol, w.SH[5], Rb);  // Q of the stack: (nbt n) x kq
  double* Q = static_cast<double*>(Qo.get(std::max<size_t>(1, size_t(rp.own) * kq) * sizeof(double)));
  if (kq == 0) return 0;
  PTB_CUDA_CHECK(cudaFuncSetAttribute(k_tsqr_apply4, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int((size_t(TS_ROWS) * TS_MAXN + TS_MAXN) * sizeof(double))));
  const int leaf0 = rp.r0 / TS_ROWS;
  const TsApply ap{V, rp.own, n, nbo, tau, static_cast<const double*>(w.SH[5].ptr) + size_t(leaf0) * n, nbt * n, kq, Q,
                   rp.own};
  launch_pdl(k_tsqr_apply4, dim3(unsigned(nbo), 1), dim3(QRR_THREADS), (size_t(TS_ROWS) * n + n) * sizeof(double), st,
             ap, ap);
  PTB_LAUNCH_CHECK(ctx);
  return kq;
}

// F and G together (update_svd's two QRs, the same shape): every leaf launch and every down-sweep
// launch covers both matrices, the stacks go through truncated_qr_pair (one launch per level, one
// host sync for both keep counts) — each matrix gets exactly tsqr_rows' arithmetic.
void tsqr_rows_pair(ProcWork& w, const RowPart& rp, const double* Af, const double* Ag, int lda, int n, double tol_f,
                    double tol_g, DeviceBuffer& Qf, DeviceBuffer& Rf, DeviceBuffer& Qg, DeviceBuffer& Rg, int& kf,
                    int& kg) {
  ptb_context* ctx = w.ctx;
  cudaStream_t st = ctx->stream;
  const int nbo = rp.own / TS_ROWS, nbt = rp.rows / TS_ROWS;
  DeviceBuffer* B[2] = {w.SH, w.SG};
  const double* A[2] = {Af, Ag};
  double *V[2], *tau[2], *So[2], *S[2];
  QrRegArgs la[2];
  for (int b = 0; b < 2; ++b) {
    V[b] = static_cast<double*>(B[b][0].get(size_t(rp.own) * n * sizeof(double)));
    tau[b] = static_cast<double*>(B[b][1].get(size_t(nbo) * n * sizeof(double)));
    So[b] = static_cast<double*>(B[b][2].get(size_t(nbo) * n * n * sizeof(double)));
    la[b] = QrRegArgs{A[b], lda, rp.own, n, nbo, 0, -1.0, nullptr, V[b], rp.own, So[b], nbo * n, tau[b], nullptr,
                      nullptr, nullptr};
  }
  launch_pdl(k_qr_reg<4, 8, false, true>, dim3(unsigned(nbo), 2), dim3(QRR_THREADS), 0, st, la[0], la[1]);
  PTB_LAUNCH_CHECK(ctx);
  for (int b = 0; b < 2; ++b) {
    S[b] = So[b];
    if (rp.W > 1) {
      S[b] = static_cast<double*>(B[b][3].get(size_t(nbt) * n * n * sizeof(double)));
      RowPart sp{rp.W, rp.rank, nbt * n, nbo * n, rp.rank * nbo * n};
      gather_rows(w, sp, So[b], n, S[b], B[b][4]);
    }
  }
  int k[2] = {0, 0};
  if (!truncated_qr_pair(w, S[0], S[1], nbt * n, n, tol_f, tol_g, w.SH[5], Rf, w.SG[5], Rg, k[0], k[1])) {
    k[0] = truncated_qr_tsqr(w, S[0], nbt * n, n, tol_f, w.SH[5], Rf);
    k[1] = truncated_qr_tsqr(w, S[1], nbt * n, n, tol_g, w.SG[5], Rg);
  }
  DeviceBuffer* Qo[2] = {&Qf, &Qg};
  TsApply ap[2];
  const int leaf0 = rp.r0 / TS_ROWS;
  for (int b = 0; b < 2; ++b) {
    double* Q = static_cast<double*>(Qo[b]->get(std::max<size_t>(1, size_t(rp.own) * k[b]) * sizeof(double)));
    ap[b] = TsApply{V[b], rp.own, n, nbo, tau[b], static_cast<const double*>(B[b][5].ptr) + size_t(leaf0) * n,
                    nbt * n, k[b], Q, rp.own};
  }
  if (k[0] > 0 || k[1] > 0) {
    PTB_CUDA_CHECK(cudaFuncSetAttribute(k_tsqr_apply4, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int((size_t(TS_ROWS) * TS_MAXN + TS_MAXN) * sizeof(double))));
    launch_pdl(k_tsqr_apply4, dim3(unsigned(nbo), 2), dim3(QRR_THREADS), (size_t(TS_ROWS) * n + n) * sizeof(double),
               st, ap[0], ap[1]);
    PTB_LAUNCH_CHECK(ctx);
  }
  kf = k[0];
  kg = k[1];
}

// PTB_QR2_PAIR=0: F and G through qr2_rows one after the other (A/B tests)
bool qr2_pair_enabled() {
  const char* e = std::getenv("PTB_QR2_PAIR");
  return !(e && std::atoi(e) == 0);
}

// the two-panel route (truncated_qr_2panel) on a row-sharded block: both panels through tsqr_rows,
// the Gram-Schmidt projections over the slabs
int qr2_rows(ProcWork& w, const RowPart& rp, const double* A, int lda, int n, double drop_tol, DeviceBuffer& Qo,
             DeviceBuffer& Rb) {
  ptb_context* ctx = w.ctx;
  cudaStream_t st = ctx->stream;
  const int n1 = TS_MAXN, n2 = n - n1, own = rp.own;
  HostProf hp_(st);
  const int k1 = tsqr_rows(w, rp, A, lda, n1, 0.0, w.TP[0], w.TP[1]);
  hp_.mark("qr2: panel 1 tsqr");
  const double* Q1 = static_cast<const double*>(w.TP[0].ptr);
  double* A2 = static_cast<double*>(w.TP[2].get(size_t(own) * n2 * sizeof(double)));
  PTB_CUDA_CHECK(cudaMemcpy2DAsync(A2, size_t(own) * sizeof(double), A + size_t(n1) * lda, size_t(lda) * sizeof(double),
                                   size_t(own) * sizeof(double), n2, cudaMemcpyDeviceToDevice, st));
  double* C = static_cast<double*>(w.TP[3].get(std::max<size_t>(1, 2 * size_t(k1) * n2) * sizeof(double)));
  if (k1 > 0) {
    for (int pass = 0; pass < 2; ++pass) {
      double* Cp = C + size_t(pass) * k1 * n2;
      slab_tn(w, rp, false, k1, n2, Q1, own, A2, own, Cp);
      gemm_rows(ctx, own, n2, k1, -1.0, Q1, own, Cp, k1, 1.0, A2, own);
    }
  }
  hp_.mark("qr2: block Gram-Schmidt x2");
  const int k2 = tsqr_rows(w, rp, A2, own, n2, 0.0, w.TP[4], w.TP[5]);
  hp_.mark("qr2: panel 2 tsqr");
  const int kk = k1 + k2;
  double* R = static_cast<double*>(w.TP[6].get(std::max<size_t>(1, size_t(kk) * n) * sizeof(double)));
  if (kk == 0) {
    Qo.get(8);
    Rb.get(8);
    return 0;
  }
  k_assemble_r2<<<unsigned(std::max(1, std::min(1024, (kk * n + 255) / 256))), 256, 0, st>>>(
      k1, k2, n1, n2, static_cast<const double*>(w.TP[1].ptr), C, C + size_t(k1) * n2,
      static_cast<const double*>(w.TP[5].ptr), R);
  PTB_LAUNCH_CHECK(ctx);
  const int kq = truncated_qr_direct(w, R, kk, n, drop_tol, w.BQ2, Rb);
  hp_.mark("qr2: R assemble + pivoted qr");
  double* Q = static_cast<double*>(Qo.get(std::max<size_t>(1, size_t(own) * kq) * sizeof(double)));
  if (kq == 0) return 0;
  const double* QR = static_cast<const double*>(w.BQ2.ptr);
  if (k1 > 0) gemm_rows(ctx, own, kq, k1, 1.0, Q1, own, QR, kk, 0.0, Q, own);
  if (k2 > 0)
    gemm_rows(ctx, own, kq, k2, 1.0, static_cast<const double*>(w.TP[4].ptr), own, QR + k1, kk, k1 > 0 ? 1.0 : 0.0, Q,
              own);
  hp_.mark("qr2: Q = [Q1 Q2] QR");
  return kq;
}

// F and G together through the two-panel route: both panels' TSQRs run as pairs (tsqr_rows_pair:
// every leaf, stack level and down-sweep launch covers both matrices, one host sync per keep-count
// pair), the Gram-Schmidt products, the R assembly + pivoted QR and the Q products per matrix —
// each matrix gets exactly qr2_rows' arithmetic.
void qr2_rows_pair(ProcWork& w, const RowPart& rp, const double* Af, const double* Ag, int lda, int n, double tol_f,
                   double tol_g, DeviceBuffer& Qf, DeviceBuffer& Rf, DeviceBuffer& Qg, DeviceBuffer& Rg, int& kf,
                   int& kg) {
  ptb_context* ctx = w.ctx;
  cudaStream_t st = ctx->stream;
  const int n1 = TS_MAXN, n2 = n - n1, own = rp.own;
  HostProf hp_(st);
  DeviceBuffer* T[2] = {w.TP, w.TPg};
  const double* A[2] = {Af, Ag};
  const double tol[2] = {tol_f, tol_g};
  DeviceBuffer* Qo[2] = {&Qf, &Qg};
  DeviceBuffer* Ro[2] = {&Rf, &Rg};
  int k1[2] = {0, 0}, k2[2] = {0, 0}, kq[2] = {0, 0};
  tsqr_rows_pair(w, rp, A[0], A[1], lda, n1, 0.0, 0.0, T[0][0], T[0][1], T[1][0], T[1][1], k1[0], k1[1]);
  hp_.mark("qr2 pair: panel 1 tsqr");
  double *A2[2], *C[2];
  for (int b = 0; b < 2; ++b) {
    const double* Q1 = static_cast<const double*>(T[b][0].ptr);
    A2[b] = static_cast<double*>(T[b][2].get(size_t(own) * n2 * sizeof(double)));
    PTB_CUDA_CHECK(cudaMemcpy2DAsync(A2[b], size_t(own) * sizeof(double), A[b] + size_t(n1) * lda,
                                     size_t(lda) * sizeof(double), size_t(own) * sizeof(double), n2,
                                     cudaMemcpyDeviceToDevice, st));
    C[b] = static_cast<double*>(T[b][3].get(std::max<size_t>(1, 2 * size_t(k1[b]) * n2) * sizeof(double)));
    if (k1[b] > 0) {
      for (int pass = 0; pass < 2; ++pass) {
        double* Cp = C[b] + size_t(pass) * k1[b] * n2;
        slab_tn(w, rp, false, k1[b], n2, Q1, own, A2[b], own, Cp);
        gemm_rows(ctx, own, n2, k1[b], -1.0, Q1, own, Cp, k1[b], 1.0, A2[b], own);
      }
    }
  }
  hp_.mark("qr2 pair: block Gram-Schmidt x2");
  tsqr_rows_pair(w, rp, A2[0], A2[1], own, n2, 0.0, 0.0, T[0][4], T[0][5], T[1][4], T[1][5], k2[0], k2[1]);
  hp_.mark("qr2 pair: panel 2 tsqr");
  for (int b = 0; b < 2; ++b) {
    const int kk = k1[b] + k2[b];
    if (kk == 0) {
      Qo[b]->get(8);
      Ro[b]->get(8);
      continue;
    }
    double* R = static_cast<double*>(T[b][6].get(std::max<size_t>(1, size_t(kk) * n) * sizeof(double)));
    k_assemble_r2<<<unsigned(std::max(1, std::min(1024, (kk * n + 255) / 256))), 256, 0, st>>>(
        k1[b], k2[b], n1, n2, static_cast<const double*>(T[b][1].ptr), C[b], C[b] + size_t(k1[b]) * n2,
        static_cast<const double*>(T[b][5].ptr), R);
    PTB_LAUNCH_CHECK(ctx);
    kq[b] = truncated_qr_direct(w, R, kk, n, tol[b], w.BQ2, *Ro[b]);
    double* Q = static_cast<double*>(Qo[b]->get(std::max<size_t>(1, size_t(own) * kq[b]) * sizeof(double)));
    if (kq[b] == 0) continue;
    const double* QR = static_cast<const double*>(w.BQ2.ptr);
    if (k1[b] > 0) gemm_rows(ctx, own, kq[b], k1[b], 1.0, static_cast<const double*>(T[b][0].ptr), own, QR, kk, 0.0, Q, own);
    if (k2[b] > 0)
      gemm_rows(ctx, own, kq[b], k2[b], 1.0, static_cast<const double*>(T[b][4].ptr), own, QR + k1[b], kk,
                k1[b] > 0 ? 1.0 : 0.0, Q, own);
  }
  hp_.mark("qr2 pair: R, pivoted qr, Q");
  kf = kq[0];
  kg = kq[1];
}

int qr_rows(ProcWork& w, const RowPart& rp, const double* A, int lda, int n, double drop_tol, DeviceBuffer& Qo,
            DeviceBuffer& Rb) {
  return n <= TS_MAXN ? tsqr_rows(w, rp, A, lda, n, drop_tol, Qo, Rb) : qr2_rows(w, rp, A, lda, n, drop_tol, Qo, Rb);
}

void update_svd_rows(ProcWork& w, DevCorrector& c, const double* F, const double* G, int rows, int cols, double tol,
                     const RowPart& rp) {
  ptb_context* ctx = w.ctx;
  cudaStream_t st = ctx->stream;
  HostProf hp_(st);
  const int r = c.rank, own = rp.own;
  const double* U = c.Xp();
  const double* V = c.Yp();
  double* UF = static_cast<double*>(w.buf[13].get(std::max<size_t>(1, size_t(r) * cols) * sizeof(double)));
  double* VG = static_cast<double*>(w.buf[14].get(std::max<size_t>(1, size_t(r) * cols) * sizeof(double)));
  slab_tn(w, rp, true, r, cols, U, rows, F, rows, UF);
  slab_tn(w, rp, true, r, cols, V, rows, G, rows, VG);
  // own rows of the projections F - U (U^T F), G - V (V^T G)
  double* Fr = static_cast<double*>(w.buf[15].get(size_t(own) * cols * sizeof(double)));
  double* Gr = static_cast<double*>(w.buf[16].get(size_t(own) * cols * sizeof(double)));
  PTB_CUDA_CHECK(cudaMemcpy2DAsync(Fr, size_t(own) * sizeof(double), F + rp.r0, size_t(rows) * sizeof(double),
                                   size_t(own) * sizeof(double), cols, cudaMemcpyDeviceToDevice, st));
  PTB_CUDA_CHECK(cudaMemcpy2DAsync(Gr, size_t(own) * sizeof(double), G + rp.r0, size_t(rows) * sizeof(double),
                                   size_t(own) * sizeof(double), cols, cudaMemcpyDeviceToDevice, st));
  if (r > 0) {
    gemm_rows(ctx, own, cols, r, -1.0, U + rp.r0, rows, UF, r, 1.0, Fr, own);
    gemm_rows(ctx, own, cols, r, -1.0, V + rp.r0, rows, VG, r, 1.0, Gr, own);
  }
  hp_.mark("update(rows): projections");
  const double qr_guard = 1e-14;
  const double fn = std::sqrt(dev_sumsq(ctx, F, size_t(rows) * cols, w.buf[11]));  // F, G are replicated
  const double gn = std::sqrt(dev_sumsq(ctx, G, size_t(rows) * cols, w.buf[11]));
  int qf = 0, qg = 0;
  if (cols <= TS_MAXN) {
    tsqr_rows_pair(w, rp, Fr, Gr, own, cols, qr_guard * fn, qr_guard * gn, w.QF, w.RF, w.QG, w.RG, qf, qg);
  } else if (qr2_pair_enabled()) {
    qr2_rows_pair(w, rp, Fr, Gr, own, cols, qr_guard * fn, qr_guard * gn, w.QF, w.RF, w.QG, w.RG, qf, qg);
  } else {
    qf = qr_rows(w, rp, Fr, own, cols, qr_guard * fn, w.QF, w.RF);
    qg = qr_rows(w, rp, Gr, own, cols, qr_guard * gn, w.QG, w.RG);
  }
  hp_.mark("update(rows): qr F, G");
  double* LB = static_cast<double*>(w.buf[17].get(std::max<size_t>(1, size_t(r + qf) * cols) * sizeof(double)));
  double* RB = static_cast<double*>(w.buf[18].get(std::max<size_t>(1, size_t(r + qg) * cols) * sizeof(double)));
  const unsigned nb = unsigned(std::max(1, std::min(1024, ((r + std::max(qf, qg)) * cols + 255) / 256)));
  k_stack_rows<<<nb, 256, 0, st>>>(UF, r, static_cast<double*>(w.RF.ptr), qf, cols, LB);
  PTB_LAUNCH_CHECK(ctx);
  k_stack_rows<<<nb, 256, 0, st>>>(VG, r, static_cast<double*>(w.RG.ptr), qg, cols, RB);
  PTB_LAUNCH_CHECK(ctx);
  const int hp = r + qf, hq = r + qg;
  double* H = static_cast<double*>(w.buf[12].get(size_t(hp) * hq * sizeof(double)));
  gemm(ctx, false, true, hp, hq, cols, 1.0, LB, hp, RB, hq, 0.0, H, hp);
  k_add_diag<<<1, 256, 0, st>>>(H, hp, static_cast<const double*>(c.Sd.ptr), r);
  PTB_LAUNCH_CHECK(ctx);
  std::vector<double> sigma;
  thin_svd(w, H, hp, hq, w.Uh, sigma, w.Vh);
  hp_.mark("update(rows): H + svd");
  const int keep = truncate_count(sigma, tol);
  double* X = static_cast<double*>(w.SX.get(std::max<size_t>(1, size_t(rows) * keep) * sizeof(double)));
  double* Y = static_cast<double*>(w.SY.get(std::max<size_t>(1, size_t(rows) * keep) * sizeof(double)));
  const double* Uh = static_cast<double*>(w.Uh.ptr);
  const double* Vh = static_cast<double*>(w.Vh.ptr);
  // own rows of the new factors, then every rank's rows gathered
  double* Xo = rp.W == 1 ? X : static_cast<double*>(w.SH[8].get(std::max<size_t>(1, size_t(own) * keep) * sizeof(double)));
  double* Yo = rp.W == 1 ? Y : static_cast<double*>(w.SH[9].get(std::max<size_t>(1, size_t(own) * keep) * sizeof(double)));
  if (keep > 0) {
    if (r > 0) {
      gemm_rows(ctx, own, keep, r, 1.0, U + rp.r0, rows, Uh, hp, 0.0, Xo, own);
      gemm_rows(ctx, own, keep, r, 1.0, V + rp.r0, rows, Vh, hq, 0.0, Yo, own);
    }
    if (qf > 0) gemm_rows(ctx, own, keep, qf, 1.0, static_cast<double*>(w.QF.ptr), own, Uh + r, hp, r > 0 ? 1.0 : 0.0, Xo, own);
    if (qg > 0) gemm_rows(ctx, own, keep, qg, 1.0, static_cast<double*>(w.QG.ptr), own, Vh + r, hq, r > 0 ? 1.0 : 0.0, Yo, own);
    gather_rows(w, rp, Xo, keep, X, w.SH[10]);
    gather_rows(w, rp, Yo, keep, Y, w.SH[11]);
  }
  hp_.mark("update(rows): rotate + gather");
  fix_signs(ctx, X, Y, rows, keep);
  sigma.resize(size_t(keep));
  PTB_CUDA_CHECK(cudaStreamSynchronize(st));
  std::swap(c.X, w.SX);
  std::swap(c.Y, w.SY);
  c.assign(rows, keep, sigma, tol);
}

void update_svd(ProcWork& w, DevCorrector& c, const double* F, const double* G, int rows, int cols, double tol) {
  check_tol(tol);
  ptb_context* ctx = w.ctx;
  if (c.empty()) {  // F, G are not read from c: solve straight into its buffers
    solve_from_scratch(w, c, F, G, rows, cols, tol);
    return;
  }
  require(rows == c.rows, "update_svd: block rows do not match corrector");
  if (RowPart rp{}; row_shard(rows, cols, w.comm, rp)) {
    update_svd_rows(w, c, F, G, rows, cols, tol, rp);
    return;
  }
  HostProf hp_(ctx->stream);
  const int r = c.rank;
  const double* U = c.Xp();
  const double* V = c.Yp();
  double* UF = static_cast<double*>(w.buf[13].get(std::max<size_t>(1, size_t(r) * cols) * sizeof(double)));
  double* VG = static_cast<double*>(w.buf[14].get(std::max<size_t>(1, size_t(r) * cols) * sizeof(double)));
  gemm(ctx, true, false, r, cols, rows, 1.0, U, rows, F, rows, 0.0, UF, r);
  gemm(ctx, true, false, r, cols, rows, 1.0, V, rows, G, rows, 0.0, VG, r);
  double* Fr = static_cast<double*>(w.buf[15].get(size_t(rows) * cols * sizeof(double)));
  double* Gr = static_cast<double*>(w.buf[16].get(size_t(rows) * cols * sizeof(double)));
  PTB_CUDA_CHECK(cudaMemcpyAsync(Fr, F, size_t(rows) * cols * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  PTB_CUDA_CHECK(cudaMemcpyAsync(Gr, G, size_t(rows) * cols * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  gemm(ctx, false, false, rows, cols, r, -1.0, U, rows, UF, r, 1.0, Fr, rows);
  gemm(ctx, false, false, rows, cols, r, -1.0, V, rows, VG, r, 1.0, Gr, rows);
  hp_.mark("update: projections");
  const double qr_guard = 1e-14;
  const double fn = std::sqrt(dev_sumsq(ctx, F, size_t(rows) * cols, w.buf[11]));
  const double gn = std::sqrt(dev_sumsq(ctx, G, size_t(rows) * cols, w.buf[11]));
  hp_.mark("update: norms");
  int qf = 0, qg = 0;
  if (truncated_qr_pair(w, Fr, Gr, rows, cols, qr_guard * fn, qr_guard * gn, w.QF, w.RF, w.QG, w.RG, qf, qg)) {
    hp_.mark("update: qr F+G (batched TSQR)");
  } else {
    qf = truncated_qr(w, Fr, rows, cols, qr_guard * fn, w.QF, w.RF);
    hp_.mark("update: qr F");
    qg = truncated_qr(w, Gr, rows, cols, qr_guard * gn, w.QG, w.RG);
    hp_.mark("update: qr G");
  }
  double* LB = static_cast<double*>(w.buf[17].get(std::max<size_t>(1, size_t(r + qf) * cols) * sizeof(double)));
  double* RB = static_cast<double*>(w.buf[18].get(std::max<size_t>(1, size_t(r + qg) * cols) * sizeof(double)));
  const unsigned nb = unsigned(std::max(1, std::min(1024, ((r + std::max(qf, qg)) * cols + 255) / 256)));
  k_stack_rows<<<nb, 256, 0, ctx->stream>>>(UF, r, static_cast<double*>(w.RF.ptr), qf, cols, LB);
  PTB_LAUNCH_CHECK(ctx);
  k_stack_rows<<<nb, 256, 0, ctx->stream>>>(VG, r, static_cast<double*>(w.RG.ptr), qg, cols, RB);
  PTB_LAUNCH_CHECK(ctx);
  const int hp = r + qf, hq = r + qg;
  double* H = static_cast<double*>(w.buf[12].get(size_t(hp) * hq * sizeof(double)));
  gemm(ctx, false, true, hp, hq, cols, 1.0, LB, hp, RB, hq, 0.0, H, hp);
  k_add_diag<<<1, 256, 0, ctx->stream>>>(H, hp, static_cast<const double*>(c.Sd.ptr), r);
  PTB_LAUNCH_CHECK(ctx);
  hp_.mark("update: H");
  std::vector<double> sigma;
  thin_svd(w, H, hp, hq, w.Uh, sigma, w.Vh);
  hp_.mark("update: svd");
  const int keep = truncate_count(sigma, tol);
  // Uext = [U QF], Vext = [V QG]; X = Uext Uh[:, :keep], Y = Vext Vh[:, :keep]
  // new factors into the spare buffers (U, V = c's factors are still read below), then swap
  double* X = static_cast<double*>(w.SX.get(std::max<size_t>(1, size_t(rows) * keep) * sizeof(double)));
  double* Y = static_cast<double*>(w.SY.get(std::max<size_t>(1, size_t(rows) * keep) * sizeof(double)));
  hp_.mark("update: alloc X/Y");
  const double* Uh = static_cast<double*>(w.Uh.ptr);
  const double* Vh = static_cast<double*>(w.Vh.ptr);
  gemm(ctx, false, false, rows, keep, r, 1.0, U, rows, Uh, hp, 0.0, X, rows);
  gemm(ctx, false, false, rows, keep, qf, 1.0, static_cast<double*>(w.QF.ptr), rows, Uh + r, hp, 1.0, X, rows);
  gemm(ctx, false, false, rows, keep, r, 1.0, V, rows, Vh, hq, 0.0, Y, rows);
  gemm(ctx, false, false, rows, keep, qg, 1.0, static_cast<double*>(w.QG.ptr), rows, Vh + r, hq, 1.0, Y, rows);
  hp_.mark("update: rotate gemms");
  fix_signs(ctx, X, Y, rows, keep);
  sigma.resize(size_t(keep));
  PTB_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  hp_.mark("update: rotate");
  std::swap(c.X, w.SX);
  std::swap(c.Y, w.SY);
  c.assign(rows, keep, sigma, tol);
  hp_.mark("update: assign");
}

// out (rows x batch) = X (Y^T in)   (procrustes.cpp:82-86)
void apply_corrector(ProcWork& w, const DevCorrector& c, size_t batch, const double* in, size_t ld_in, double* out,
                     size_t ld_out) {
  ptb_context* ctx = w.ctx;
  if (batch == 0) return;
  if (c.rank == 0) {
    PTB_CUDA_CHECK(cudaMemset2DAsync(out, ld_out * sizeof(double), 0, size_t(c.rows) * sizeof(double), batch,
                                     ctx->stream));
    return;
  }
  double* z = static_cast<double*>(w.buf[19].get(size_t(c.rank) * batch * sizeof(double)));
  gemm(ctx, true, false, c.rank, int(batch), c.rows, 1.0, c.Yp(), c.rows, in, int(ld_in), 0.0, z, c.rank);
  gemm(ctx, false, false, c.rows, int(batch), c.rank, 1.0, c.Xp(), c.rows, z, c.rank, 0.0, out, int(ld_out));
}

// procrustes.cpp:245-253
double relative_residual(ProcWork& w, const DevCorrector& c, const double* F, const double* G, int rows, int cols) {
  ptb_context* ctx = w.ctx;
  const double fnorm = std::sqrt(dev_sumsq(ctx, F, size_t(rows) * cols, w.buf[11]));
  if (fnorm == 0.0) return 0.0;
  if (c.rank == 0) return 1.0;
  double* D = static_cast<double*>(w.buf[20].get(size_t(rows) * cols * sizeof(double)));
  apply_corrector(w, c, size_t(cols), G, size_t(rows), D, size_t(rows));
  // D = F - X Y^T G
  geam_sub(ctx, size_t(rows) * cols, F, D);
  return std::sqrt(dev_sumsq(ctx, D, size_t(rows) * cols, w.buf[11])) / fnorm;
}

void drop_leading(const DevCorrector& c, size_t count, DevCorrector& out, ptb_context* ctx) {
  const int keep = std::max(0, c.rank - int(std::min<size_t>(count, size_t(c.rank))));
  const int first = c.rank - keep;
  double* X = static_cast<double*>(out.X.get(std::max<size_t>(1, size_t(c.rows) * keep) * sizeof(double)));
  double* Y = static_cast<double*>(out.Y.get(std::max<size_t>(1, size_t(c.rows) * keep) * sizeof(double)));
  if (keep > 0) {
    PTB_CUDA_CHECK(cudaMemcpyAsync(X, c.Xp() + size_t(first) * c.rows, size_t(c.rows) * keep * sizeof(double),
                                   cudaMemcpyDeviceToDevice, ctx->stream));
    PTB_CUDA_CHECK(cudaMemcpyAsync(Y, c.Yp() + size_t(first) * c.rows, size_t(c.rows) * keep * sizeof(double),
                                   cudaMemcpyDeviceToDevice, ctx->stream));
  }
  PTB_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
  out.assign(c.rows, keep, std::vector<double>(c.S.begin() + first, c.S.end()), c.tol);
}

}  // namespace ptb

