// PhaseCorrector text checkpoint on the drop-in API (procrustes.hpp:41-43, procrustes.cpp:95-127),
// mirroring the reference's "checkpoint text round trip" case (test_procrustes.cpp:209-224),
// which itself cannot be compiled here because it is written against Eigen.  Host-only: the
// checkpoint is plain text I/O, so this suite runs in the CPU test tier.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"

#include <cmath>
#include <random>
#include <sstream>
#include <stdexcept>

#include "paratime/procrustes.hpp"

using namespace paratime;

namespace {
Matrix random_matrix(Index rows, Index cols, std::mt19937_64& rng) {
  std::normal_distribution<double> d(0.0, 1.0);
  Matrix m(rows, cols);
  for (Index j = 0; j < cols; ++j)
    for (Index i = 0; i < rows; ++i) m(i, j) = d(rng);
  return m;
}
double max_abs_diff(const Matrix& a, const Matrix& b) {
  double m = 0.0;
  for (Index k = 0; k < a.rows() * a.cols(); ++k) m = std::max(m, std::abs(a.data()[k] - b.data()[k]));
  return m;
}
}  // namespace

TEST_CASE("checkpoint text round trip (host factors)") {
  std::mt19937_64 rng(151);
  const Matrix X = random_matrix(14, 4, rng), Y = random_matrix(14, 4, rng);
  const PhaseCorrector c(X, {3.5, 1.25, 1e-7, 4.9e-300}, Y, 1e-13);
  std::stringstream ss;
  c.save(ss);
  const PhaseCorrector back = PhaseCorrector::load(ss);
  REQUIRE(back.rank() == c.rank());
  REQUIRE(back.rows() == c.rows());
  CHECK(max_abs_diff(back.left(), c.left()) == 0.0);  // 17 significant digits round-trip exactly
  CHECK(max_abs_diff(back.right(), c.right()) == 0.0);
  for (Index i = 0; i < c.rank(); ++i) CHECK(back.singular_values()[size_t(i)] == c.singular_values()[size_t(i)]);
  CHECK(back.tol() == 0.0);  // procrustes.cpp:126: loaded correctors carry tol 0
}

TEST_CASE("checkpoint header and layout follow procrustes.cpp:95-108") {
  Matrix X(2, 1), Y(2, 1);
  X(0, 0) = 0.5;
  X(1, 0) = -2.0;
  Y(0, 0) = 1.0;
  Y(1, 0) = 0.1;
  std::stringstream ss;
  PhaseCorrector(X, {3.0}, Y, 1e-8).save(ss);
  CHECK(ss.str() == "2 1\n0.5\n-2\n3\n1\n0.10000000000000001\n");
}

TEST_CASE("empty corrector round trips") {
  std::stringstream ss;
  PhaseCorrector().save(ss);
  const PhaseCorrector back = PhaseCorrector::load(ss);
  CHECK(back.rank() == 0);
  CHECK(back.rows() == 0);
}

TEST_CASE("malformed checkpoints throw runtime_error") {
  std::stringstream bad("3 junk");
  CHECK_THROWS_AS(PhaseCorrector::load(bad), std::runtime_error);
  std::stringstream trunc("2 1\n0.5\n");
  CHECK_THROWS_AS(PhaseCorrector::load(trunc), std::runtime_error);
}
