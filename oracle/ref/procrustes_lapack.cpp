// ORACLE — test infrastructure only (tests/, bench.py cpu_baseline, smoke()).
//
// Restatement of /root/reference/proj/src/procrustes.cpp on LAPACK, because the
// reference's Eigen3 dependency is absent from this image.  Line references are to
// that file.  Third-party mapping (Eigen3 >= 3.3, unpinned, CMakeLists.txt:13):
//   Eigen::ColPivHouseholderQR   -> dgeqp3 + dorgqr   (same column-pivoting rule)
//   Eigen::BDCSVD (thin U, V)    -> dgesdd jobz='S'
//   Eigen GEMM products          -> dgemm
// LAPACK comes from scipy's bundled OpenBLAS (LP64, symbols prefixed scipy_).

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <vector>

#include "paratime/procrustes.hpp"

extern "C" {
void scipy_dgeqp3_(const int* m, const int* n, double* a, const int* lda, int* jpvt, double* tau,
                   double* work, const int* lwork, int* info);
void scipy_dorgqr_(const int* m, const int* n, const int* k, double* a, const int* lda,
                   const double* tau, double* work, const int* lwork, int* info);
void scipy_dgesdd_(const char* jobz, const int* m, const int* n, double* a, const int* lda,
                   double* s, double* u, const int* ldu, double* vt, const int* ldvt, double* work,
                   const int* lwork, int* iwork, int* info);
void scipy_dgemm_(const char* ta, const char* tb, const int* m, const int* n, const int* k,
                  const double* alpha, const double* a, const int* lda, const double* b,
                  const int* ldb, const double* beta, double* c, const int* ldc);
}

namespace paratime {

double OMat::squaredNorm() const {
  double acc = 0.0;
  for (double v : data_) acc += v * v;
  return acc;
}

double OMat::norm() const { return std::sqrt(squaredNorm()); }

OMat operator-(const OMat& a, const OMat& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols())
    throw std::invalid_argument("OMat: shape mismatch in subtraction");
  OMat out(a.rows(), a.cols());
  for (OIndex j = 0; j < a.cols(); ++j)
    for (OIndex i = 0; i < a.rows(); ++i) out(i, j) = a(i, j) - b(i, j);
  return out;
}

namespace {

// C = op(A) * op(B)
OMat gemm(const OMat& A, bool ta, const OMat& B, bool tb) {
  const int m = static_cast<int>(ta ? A.cols() : A.rows());
  const int k = static_cast<int>(ta ? A.rows() : A.cols());
  const int n = static_cast<int>(tb ? B.rows() : B.cols());
  const int kb = static_cast<int>(tb ? B.cols() : B.rows());
  if (k != kb) throw std::invalid_argument("gemm: inner dimension mismatch");
  OMat C(m, n);
  if (m == 0 || n == 0) return C;
  if (k == 0) return C;
  const char cta = ta ? 'T' : 'N', ctb = tb ? 'T' : 'N';
  const double one = 1.0, zero = 0.0;
  const int lda = std::max<int>(1, static_cast<int>(A.rows()));
  const int ldb = std::max<int>(1, static_cast<int>(B.rows()));
  const int ldc = std::max(1, m);
  scipy_dgemm_(&cta, &ctb, &m, &n, &k, &one, A.data(), &lda, B.data(), &ldb, &zero, C.data(),
               &ldc);
  return C;
}

OMat left_cols(const OMat& A, OIndex count) {
  OMat out(A.rows(), count);
  std::copy(A.data(), A.data() + A.rows() * count, out.data());
  return out;
}

// procrustes.cpp:14-17
void check_tol(double tol) {
  if (!(tol > 0.0) || !(tol < 1.0))
    throw std::invalid_argument("truncation tolerance must lie in (0, 1)");
}

// procrustes.cpp:21-30 — largest-magnitude entry of each left column made
// positive (first maximum on ties, as Eigen's maxCoeff), right column flipped too.
void fix_signs(OMat& left, OMat& right) {
  for (OIndex j = 0; j < left.cols(); ++j) {
    OIndex imax = 0;
    double best = -1.0;
    for (OIndex i = 0; i < left.rows(); ++i) {
      const double a = std::abs(left(i, j));
      if (a > best) {
        best = a;
        imax = i;
      }
    }
    if (left.rows() > 0 && left(imax, j) < 0.0) {
      for (OIndex i = 0; i < left.rows(); ++i) left(i, j) = -left(i, j);
      for (OIndex i = 0; i < right.rows(); ++i) right(i, j) = -right(i, j);
    }
  }
}

// procrustes.cpp:34-46 — column-pivoted thin QR, R un-pivoted (R P^T), keep
// the leading pivoted diagonal entries whose magnitude exceeds drop_tol.
void truncated_qr(const OMat& A, double drop_tol, OMat& Q, OMat& R) {
  const int m = static_cast<int>(A.rows()), n = static_cast<int>(A.cols());
  const int k = std::min(m, n);
  if (k == 0) {
    Q = OMat(A.rows(), 0);
    R = OMat(0, A.cols());
    return;
  }
  OMat work_a = A;
  std::vector<int> jpvt(static_cast<std::size_t>(n), 0);
  std::vector<double> tau(static_cast<std::size_t>(k));
  int info = 0, lwork = -1;
  double wq = 0.0;
  scipy_dgeqp3_(&m, &n, work_a.data(), &m, jpvt.data(), tau.data(), &wq, &lwork, &info);
  lwork = std::max(1, static_cast<int>(wq));
  std::vector<double> work(static_cast<std::size_t>(lwork));
  scipy_dgeqp3_(&m, &n, work_a.data(), &m, jpvt.data(), tau.data(), work.data(), &lwork, &info);
  if (info != 0) throw std::runtime_error("dgeqp3 failed");

  OIndex keep = 0;
  while (keep < k && std::abs(work_a(keep, keep)) > drop_tol) ++keep;

  R = OMat(keep, n);
  for (int j = 0; j < n; ++j) {
    const int orig = jpvt[static_cast<std::size_t>(j)] - 1;
    for (OIndex i = 0; i < keep && i <= j; ++i) R(i, orig) = work_a(i, j);
  }

  OMat q = left_cols(work_a, k);
  lwork = -1;
  scipy_dorgqr_(&m, &k, &k, q.data(), &m, tau.data(), &wq, &lwork, &info);
  lwork = std::max(1, static_cast<int>(wq));
  work.assign(static_cast<std::size_t>(lwork), 0.0);
  scipy_dorgqr_(&m, &k, &k, q.data(), &m, tau.data(), work.data(), &lwork, &info);
  if (info != 0) throw std::runtime_error("dorgqr failed");
  Q = left_cols(q, keep);
}

// thin SVD, singular values descending: M = U diag(s) V^T
void thin_svd(const OMat& M, OMat& U, std::vector<double>& s, OMat& V) {
  const int m = static_cast<int>(M.rows()), n = static_cast<int>(M.cols());
  const int k = std::min(m, n);
  s.assign(static_cast<std::size_t>(k), 0.0);
  U = OMat(m, k);
  V = OMat(n, k);
  if (k == 0) return;
  OMat a = M;
  OMat vt(k, n);
  const char jobz = 'S';
  int info = 0, lwork = -1;
  double wq = 0.0;
  std::vector<int> iwork(static_cast<std::size_t>(8 * k));
  const int ldvt = k;
  scipy_dgesdd_(&jobz, &m, &n, a.data(), &m, s.data(), U.data(), &m, vt.data(), &ldvt, &wq,
                &lwork, iwork.data(), &info);
  lwork = std::max(1, static_cast<int>(wq));
  std::vector<double> work(static_cast<std::size_t>(lwork));
  scipy_dgesdd_(&jobz, &m, &n, a.data(), &m, s.data(), U.data(), &m, vt.data(), &ldvt,
                work.data(), &lwork, iwork.data(), &info);
  if (info != 0) throw std::runtime_error("dgesdd failed");
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < n; ++j) V(j, i) = vt(i, j);
}

// procrustes.cpp:48-69
PhaseCorrector solve_from_scratch(const SnapshotMatrix& F, const SnapshotMatrix& G, double tol) {
  const double qr_guard = 1e-14;
  OMat QF, RF, QG, RG;
  truncated_qr(F, qr_guard * F.norm(), QF, RF);
  truncated_qr(G, qr_guard * G.norm(), QG, RG);
  if (QF.cols() == 0 || QG.cols() == 0)
    return PhaseCorrector(OMat(F.rows(), 0), {}, OMat(F.rows(), 0), tol);

  OMat U, V;
  std::vector<double> sigma;
  thin_svd(gemm(RF, false, RG, true), U, sigma, V);
  const double smax = sigma.empty() ? 0.0 : sigma[0];
  OIndex s = 0;
  while (s < static_cast<OIndex>(sigma.size()) && smax > 0.0 && sigma[static_cast<std::size_t>(s)] / smax > tol) ++s;

  OMat X = gemm(QF, false, left_cols(U, s), false);
  OMat Y = gemm(QG, false, left_cols(V, s), false);
  fix_signs(X, Y);
  sigma.resize(static_cast<std::size_t>(s));
  return PhaseCorrector(std::move(X), std::move(sigma), std::move(Y), tol);
}

}  // namespace

PhaseCorrector::PhaseCorrector(OMat left, std::vector<double> singular_values, OMat right,
                               double tol)
    : left_(std::move(left)), sv_(std::move(singular_values)), right_(std::move(right)),
      tol_(tol) {
  if (left_.rows() != right_.rows() || left_.cols() != right_.cols() ||
      left_.cols() != static_cast<OIndex>(sv_.size()))
    throw std::invalid_argument("PhaseCorrector: inconsistent factor shapes");
}

// procrustes.cpp:82-86
std::vector<double> PhaseCorrector::apply(const std::vector<double>& stacked) const {
  if (static_cast<OIndex>(stacked.size()) != rows())
    throw std::invalid_argument("PhaseCorrector: stacked length does not match rows");
  OMat v(rows(), 1);
  std::copy(stacked.begin(), stacked.end(), v.data());
  const OMat z = gemm(right_, true, v, false);
  const OMat out = gemm(left_, false, z, false);
  return std::vector<double>(out.data(), out.data() + out.rows());
}

// procrustes.cpp:88-93
PhaseCorrector PhaseCorrector::drop_leading(OIndex count) const {
  if (count < 0) throw std::invalid_argument("drop_leading: negative count");
  const OIndex keep = std::max<OIndex>(0, rank() - count);
  const OIndex first = rank() - keep;
  OMat l(rows(), keep), r(rows(), keep);
  std::copy(left_.col(first), left_.col(first) + rows() * keep, l.data());
  std::copy(right_.col(first), right_.col(first) + rows() * keep, r.data());
  std::vector<double> sv(sv_.begin() + first, sv_.end());
  return PhaseCorrector(std::move(l), std::move(sv), std::move(r), tol_);
}

// procrustes.cpp:129-142
std::vector<double> stack_components(const EnergyComponents& comp) {
  std::vector<double> out;
  out.reserve((comp.grad.size() + 1) * comp.grid.size());
  for (const auto& block : comp.grad) out.insert(out.end(), block.begin(), block.end());
  out.insert(out.end(), comp.momentum.begin(), comp.momentum.end());
  return out;
}

// procrustes.cpp:144-156
EnergyComponents unstack_components(const std::vector<double>& stacked, const Grid& grid,
                                    double mean_u) {
  const std::size_t n = grid.size();
  const std::size_t d = static_cast<std::size_t>(grid.dim());
  if (stacked.size() != (d + 1) * n)
    throw std::invalid_argument("unstack_components: length does not match grid");
  EnergyComponents comp{grid, {}, std::vector<double>(n), mean_u};
  std::size_t at = 0;
  for (std::size_t a = 0; a < d; ++a) {
    comp.grad.emplace_back(stacked.begin() + static_cast<long>(at),
                           stacked.begin() + static_cast<long>(at + n));
    at += n;
  }
  std::copy(stacked.begin() + static_cast<long>(at), stacked.end(), comp.momentum.begin());
  return comp;
}

// procrustes.cpp:158-175
std::pair<SnapshotMatrix, SnapshotMatrix> assemble_snapshots(
    std::span<const WaveState> fine_states, std::span<const WaveState> coarse_states,
    const GridTransfer& transfer, const SpeedField& coarse_speed, GradientScheme scheme) {
  if (fine_states.empty() || fine_states.size() != coarse_states.size())
    throw std::invalid_argument("assemble_snapshots: need equal, nonempty snapshot lists");
  const OIndex rows = static_cast<OIndex>((transfer.coarse.dim() + 1) * transfer.coarse.size());
  const OIndex cols = static_cast<OIndex>(fine_states.size());
  SnapshotMatrix F(rows, cols), G(rows, cols);
  for (OIndex n = 0; n < cols; ++n) {
    const WaveState restricted = restrict_state(fine_states[static_cast<std::size_t>(n)], transfer);
    const std::vector<double> f =
        stack_components(to_energy_components(restricted, coarse_speed, scheme));
    const std::vector<double> g = stack_components(
        to_energy_components(coarse_states[static_cast<std::size_t>(n)], coarse_speed, scheme));
    std::copy(f.begin(), f.end(), F.col(n));
    std::copy(g.begin(), g.end(), G.col(n));
  }
  return {std::move(F), std::move(G)};
}

// procrustes.cpp:177-186
PhaseCorrector procrustes_solve(const SnapshotMatrix& F, const SnapshotMatrix& G, double tol) {
  check_tol(tol);
  if (F.rows() != G.rows() || F.cols() != G.cols())
    throw std::invalid_argument("procrustes_solve: F and G must have the same shape");
  if (F.cols() > F.rows())
    throw std::invalid_argument("procrustes_solve: more snapshots than rows");
  if (F.cols() == 0) throw std::invalid_argument("procrustes_solve: empty data");
  return solve_from_scratch(F, G, tol);
}

// procrustes.cpp:188-237 (Algorithm 1)
PhaseCorrector update_svd(const PhaseCorrector& corrector, const SnapshotMatrix& F,
                          const SnapshotMatrix& G, double tol) {
  check_tol(tol);
  if (F.rows() != G.rows() || F.cols() != G.cols())
    throw std::invalid_argument("update_svd: F and G must have the same shape");
  if (corrector.empty()) return solve_from_scratch(F, G, tol);
  if (F.rows() != corrector.rows())
    throw std::invalid_argument("update_svd: block rows do not match corrector");

  const OMat& U = corrector.left();
  const OMat& V = corrector.right();
  const OIndex r = corrector.rank();
  const OIndex rows = corrector.rows();

  const OMat UF = gemm(U, true, F, false);  // r x N
  const OMat VG = gemm(V, true, G, false);

  const double qr_guard = 1e-14;
  OMat QF, RF, QG, RG;
  truncated_qr(F - gemm(U, false, UF, false), qr_guard * F.norm(), QF, RF);
  truncated_qr(G - gemm(V, false, VG, false), qr_guard * G.norm(), QG, RG);
  const OIndex qf = QF.cols(), qg = QG.cols();

  OMat left_block(r + qf, F.cols()), right_block(r + qg, G.cols());
  for (OIndex j = 0; j < F.cols(); ++j) {
    for (OIndex i = 0; i < r; ++i) left_block(i, j) = UF(i, j);
    for (OIndex i = 0; i < qf; ++i) left_block(r + i, j) = RF(i, j);
    for (OIndex i = 0; i < r; ++i) right_block(i, j) = VG(i, j);
    for (OIndex i = 0; i < qg; ++i) right_block(r + i, j) = RG(i, j);
  }
  OMat H = gemm(left_block, false, right_block, true);
  for (OIndex i = 0; i < r; ++i) H(i, i) += corrector.singular_values()[static_cast<std::size_t>(i)];

  OMat Uh, Vh;
  std::vector<double> sigma;
  thin_svd(H, Uh, sigma, Vh);
  const double smax = sigma.empty() ? 0.0 : sigma[0];
  OIndex keep = 0;
  while (keep < static_cast<OIndex>(sigma.size()) && smax > 0.0 &&
         sigma[static_cast<std::size_t>(keep)] / smax > tol)
    ++keep;

  OMat Uext(rows, r + qf), Vext(rows, r + qg);
  std::copy(U.data(), U.data() + rows * r, Uext.data());
  std::copy(QF.data(), QF.data() + rows * qf, Uext.col(r));
  std::copy(V.data(), V.data() + rows * r, Vext.data());
  std::copy(QG.data(), QG.data() + rows * qg, Vext.col(r));

  OMat Xnew = gemm(Uext, false, left_cols(Uh, keep), false);
  OMat Ynew = gemm(Vext, false, left_cols(Vh, keep), false);
  fix_signs(Xnew, Ynew);
  sigma.resize(static_cast<std::size_t>(keep));
  return PhaseCorrector(std::move(Xnew), std::move(sigma), std::move(Ynew), tol);
}

// procrustes.cpp:239-243
EnergyComponents apply_corrector(const PhaseCorrector& corrector, const EnergyComponents& comp) {
  const std::vector<double> corrected = corrector.apply(stack_components(comp));
  return unstack_components(corrected, comp.grid, comp.mean_u);
}

// procrustes.cpp:245-253
double relative_residual(const PhaseCorrector& corrector, const SnapshotMatrix& F,
                         const SnapshotMatrix& G) {
  const double fnorm = F.norm();
  if (fnorm == 0.0) return 0.0;
  if (corrector.rank() == 0) return 1.0;
  const OMat corrected = gemm(corrector.left(), false, gemm(corrector.right(), true, G, false), false);
  return (F - corrected).norm() / fnorm;
}

}  // namespace paratime
