// Speed-model file ingestion on the drop-in API (experiment.hpp:86-90): path-based reading,
// bilinear resampling onto a target grid (grid.cpp:264-298), and the ConfigError cases of
// experiment.cpp:755-770.  Host-only (CPU tier); the text format itself is pinned against the
// reference in tests/test_speed_model.py.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"

#include <cstdio>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "paratime/errors.hpp"
#include "paratime/grid.hpp"
#include "paratime/speed_model.hpp"

using namespace paratime;

namespace {
std::string temp_path(const char* name) { return std::string("/tmp/ptb_") + name + ".txt"; }

SpeedField sample_field() {
  std::vector<double> c(6 * 5);
  for (std::size_t i = 0; i < c.size(); ++i) c[i] = 1.0 + 0.1 * double(i % 7) + 0.01 * double(i);
  return SpeedField(Grid({6, 5}, {1.0 / 6, 0.2}), c);
}
}  // namespace

TEST_CASE("ingest_speed_model reads what write_speed_model wrote") {
  const SpeedField f = sample_field();
  const std::string p = temp_path("sm_roundtrip");
  {
    std::ofstream os(p);
    write_speed_model(f, os);
  }
  const SpeedField g = ingest_speed_model(p);
  REQUIRE(g.grid.dim() == 2);
  CHECK(g.grid.points(0) == 6);
  CHECK(g.grid.points(1) == 5);
  CHECK(g.c == f.c);
  std::remove(p.c_str());
}

TEST_CASE("ingest onto a target grid is the bilinear resample of the file") {
  const SpeedField f = sample_field();
  const std::string p = temp_path("sm_resample");
  {
    std::ofstream os(p);
    write_speed_model(f, os);
  }
  const Grid target({12, 10}, {1.0 / 12, 0.1});
  const SpeedField g = ingest_speed_model(p, target);
  CHECK(g.c == bilinear_resample(f.c, 6, 5, 12, 10));
  CHECK_THROWS_AS(ingest_speed_model(p, Grid({3, 4}, {0.1, 0.1})), std::invalid_argument);  // Grid: >= 4 points
  std::remove(p.c_str());
}

TEST_CASE("ingestion errors are ConfigError") {
  CHECK_THROWS_AS(ingest_speed_model("/nonexistent/speed.txt"), ConfigError);
  const std::string p = temp_path("sm_1d");
  {
    std::ofstream os(p);
    os << "1 6 1 0.2\n1 2 3 4 5 6\n";
  }
  CHECK(ingest_speed_model(p).grid.dim() == 1);
  CHECK_THROWS_AS(ingest_speed_model(p, Grid({8, 8}, {0.125, 0.125})), ConfigError);  // 1D file, 2D grid
  std::remove(p.c_str());
}
