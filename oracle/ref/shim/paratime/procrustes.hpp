#pragma once
// ORACLE SHIM — test infrastructure only (tests/, bench.py cpu_baseline, smoke()).
//
// Stands in for /root/reference/proj/include/paratime/procrustes.hpp so that the
// reference's parareal.cpp / experiment.cpp compile verbatim in oracle/_ref.  The
// reference header types SnapshotMatrix as Eigen::MatrixXd (procrustes.hpp:16) and
// Eigen3 is not installed in this image, so the factor storage becomes the small
// column-major OMat below.  Every member parareal.cpp:249-308 touches is provided
// with the same meaning: norm() (Frobenius), operator-, rows(), cols().
// The algorithms behind these declarations are restated in procrustes_lapack.cpp
// on top of LAPACK (dgeqp3/dorgqr/dgesdd) from the bundled scipy-openblas.

#include <cstddef>
#include <iosfwd>
#include <span>
#include <utility>
#include <vector>

#include "paratime/energy_map.hpp"
#include "paratime/grid.hpp"

namespace paratime {

using OIndex = long;

/// Column-major dense matrix (the oracle's stand-in for Eigen::MatrixXd).
class OMat {
 public:
  OMat() = default;
  OMat(OIndex rows, OIndex cols, double fill = 0.0)
      : rows_(rows), cols_(cols), data_(static_cast<std::size_t>(rows * cols), fill) {}

  OIndex rows() const { return rows_; }
  OIndex cols() const { return cols_; }
  double& operator()(OIndex i, OIndex j) { return data_[static_cast<std::size_t>(j * rows_ + i)]; }
  double operator()(OIndex i, OIndex j) const {
    return data_[static_cast<std::size_t>(j * rows_ + i)];
  }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }
  double* col(OIndex j) { return data_.data() + j * rows_; }
  const double* col(OIndex j) const { return data_.data() + j * rows_; }

  double squaredNorm() const;
  double norm() const;  // Frobenius, as Eigen::MatrixBase::norm()

 private:
  OIndex rows_ = 0, cols_ = 0;
  std::vector<double> data_;
};

OMat operator-(const OMat& a, const OMat& b);

using SnapshotMatrix = OMat;

class PhaseCorrector {
 public:
  PhaseCorrector() = default;
  PhaseCorrector(OMat left, std::vector<double> singular_values, OMat right, double tol);

  bool empty() const { return left_.rows() == 0; }
  OIndex rows() const { return left_.rows(); }
  OIndex rank() const { return static_cast<OIndex>(sv_.size()); }
  const OMat& left() const { return left_; }
  const OMat& right() const { return right_; }
  const std::vector<double>& singular_values() const { return sv_; }
  double tol() const { return tol_; }

  std::vector<double> apply(const std::vector<double>& stacked) const;
  PhaseCorrector drop_leading(OIndex count) const;

 private:
  OMat left_;
  std::vector<double> sv_;
  OMat right_;
  double tol_ = 0.0;
};

std::vector<double> stack_components(const EnergyComponents& comp);
EnergyComponents unstack_components(const std::vector<double>& stacked, const Grid& grid,
                                    double mean_u);

std::pair<SnapshotMatrix, SnapshotMatrix> assemble_snapshots(
    std::span<const WaveState> fine_states, std::span<const WaveState> coarse_states,
    const GridTransfer& transfer, const SpeedField& coarse_speed, GradientScheme scheme);

PhaseCorrector procrustes_solve(const SnapshotMatrix& F, const SnapshotMatrix& G, double tol);
PhaseCorrector update_svd(const PhaseCorrector& corrector, const SnapshotMatrix& F,
                          const SnapshotMatrix& G, double tol);
EnergyComponents apply_corrector(const PhaseCorrector& corrector, const EnergyComponents& comp);
double relative_residual(const PhaseCorrector& corrector, const SnapshotMatrix& F,
                         const SnapshotMatrix& G);

}  // namespace paratime
