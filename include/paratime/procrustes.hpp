// paratime_b200 drop-in for /root/reference/proj/include/paratime/procrustes.hpp:16-81.
// Forced deviation: SnapshotMatrix is Eigen::MatrixXd in the reference;
// Eigen is not part of this build, so it is the column-major paratime::Matrix below, which
// provides the members the reference's driver uses (rows, cols, norm, operator-).
#pragma once

#include <cstddef>
#include <iosfwd>
#include <span>
#include <utility>
#include <vector>

#include "paratime/energy_map.hpp"
#include "paratime/grid.hpp"

namespace paratime {

using Index = long;

/// Dense column-major matrix.
class Matrix {
 public:
  Matrix() = default;
  Matrix(Index rows, Index cols, double fill = 0.0)
      : rows_(rows), cols_(cols), data_(static_cast<std::size_t>(rows * cols), fill) {}
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  double& operator()(Index i, Index j) { return data_[static_cast<std::size_t>(j * rows_ + i)]; }
  double operator()(Index i, Index j) const { return data_[static_cast<std::size_t>(j * rows_ + i)]; }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }
  double* col(Index j) { return data_.data() + j * rows_; }
  const double* col(Index j) const { return data_.data() + j * rows_; }
  double squaredNorm() const;
  double norm() const;  // Frobenius

 private:
  Index rows_ = 0, cols_ = 0;
  std::vector<double> data_;
};

Matrix operator-(const Matrix& a, const Matrix& b);
Matrix operator+(const Matrix& a, const Matrix& b);

using SnapshotMatrix = Matrix;

/// Truncated factors (X, S, Y) of M = sum_k F_k G_k^T; acts as v -> X (Y^T v).
class PhaseCorrector {
 public:
  PhaseCorrector() = default;
  PhaseCorrector(Matrix left, std::vector<double> singular_values, Matrix right, double tol);

  bool empty() const { return left_.rows() == 0; }
  Index rows() const { return left_.rows(); }
  Index rank() const { return static_cast<Index>(sv_.size()); }
  const Matrix& left() const { return left_; }
  const Matrix& right() const { return right_; }
  const std::vector<double>& singular_values() const { return sv_; }
  double tol() const { return tol_; }

  std::vector<double> apply(const std::vector<double>& stacked) const;
  PhaseCorrector drop_leading(Index count) const;

  /// Text checkpoint: "rows r" header then X, S, Y blocks (procrustes.hpp:41-43).
  void save(std::ostream& os) const;
  static PhaseCorrector load(std::istream& is);

 private:
  Matrix left_;
  std::vector<double> sv_;
  Matrix right_;
  double tol_ = 0.0;
};

std::vector<double> stack_components(const EnergyComponents& comp);
EnergyComponents unstack_components(const std::vector<double>& stacked, const Grid& grid, double mean_u);

std::pair<SnapshotMatrix, SnapshotMatrix> assemble_snapshots(std::span<const WaveState> fine_states,
                                                             std::span<const WaveState> coarse_states,
                                                             const GridTransfer& transfer,
                                                             const SpeedField& coarse_speed, GradientScheme scheme);
PhaseCorrector procrustes_solve(const SnapshotMatrix& F, const SnapshotMatrix& G, double tol);
PhaseCorrector update_svd(const PhaseCorrector& corrector, const SnapshotMatrix& F, const SnapshotMatrix& G,
                          double tol);
EnergyComponents apply_corrector(const PhaseCorrector& corrector, const EnergyComponents& comp);
double relative_residual(const PhaseCorrector& corrector, const SnapshotMatrix& F, const SnapshotMatrix& G);

}  // namespace paratime
