// Absorbing-layer extension of the drop-in API (include/paratime/pml.hpp) on the B200: the
// reference has no layer, so the pins are self-consistency ones in the reference's test style
// (test_propagator.cpp): zero damping = propagate_coupling (fast mode) bitwise, batch = single,
// PropagationDiverged / std::invalid_argument like PropagatorConfig.  Runs on the GPU box
// (tests/test_gpu_pml.py).
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"

#include <cmath>
#include <limits>
#include <stdexcept>
#include <vector>

#include "paratime/errors.hpp"
#include "paratime/parareal.hpp"
#include "paratime/grid.hpp"
#include "paratime/pml.hpp"
#include "paratime/propagator.hpp"

using namespace paratime;

namespace {
Grid grid2(std::size_t n) { return Grid({n, n}, {1.0 / double(n), 1.0 / double(n)}); }

WaveState pulse(const Grid& g) {
  const std::size_t n = g.points(0);
  std::vector<double> u(g.size());
  for (std::size_t iy = 0; iy < n; ++iy)
    for (std::size_t ix = 0; ix < n; ++ix) {
      const double x = double(ix) / double(n) - 0.5, y = double(iy) / double(n) - 0.45;
      u[iy * n + ix] = std::exp(-300.0 * (x * x + y * y));
    }
  return WaveState(g, u, std::vector<double>(g.size(), 0.0));
}
}  // namespace

TEST_CASE("zero damping reproduces propagate_coupling (fast mode) bitwise") {
  set_propagator_mode(PropagatorMode::fast);
  const Grid g = grid2(96);
  std::vector<double> c(g.size());
  for (std::size_t i = 0; i < c.size(); ++i) c[i] = 0.6 + 0.3 * std::sin(0.01 * double(i));
  const SpeedField s(g, c);
  const double dt = 1.0 / (96.0 * 8.0);
  const PropagatorConfig per(g, s, dt, 24);
  const PmlConfig pml(g, s, std::vector<double>(96, 0.0), std::vector<double>(96, 0.0), dt, 24);
  const WaveState w = pulse(g);
  const WaveState a = propagate_coupling(w, per);
  const PmlState b = pml_propagate_coupling(PmlState(w), pml);
  CHECK(a.u == b.wave.u);
  CHECK(a.udot == b.wave.udot);
  CHECK(b.px == std::vector<double>(g.size(), 0.0));
}

TEST_CASE("batched layered propagation equals one state at a time") {
  const Grid g = grid2(80);
  const SpeedField s(g, std::vector<double>(g.size(), 1.0));
  const auto z = pml_damping_profile(80, 10, 1.0 / 80, 1.0);
  const PmlConfig cfg(g, s, z, z, 1.0 / 640, 16);
  std::vector<PmlState> batch{PmlState(pulse(g)), PmlState(2.0 * pulse(g))};
  const PmlState one = pml_propagate_coupling(batch[1], cfg);
  std::vector<bool> div;
  pml_propagate_coupling_batch(batch, cfg, &div);
  CHECK_FALSE(div[1]);
  CHECK(batch[1].wave.u == one.wave.u);
  CHECK(batch[1].px == one.px);
}

TEST_CASE("the layer absorbs: energy left in the box decays") {
  const Grid g = grid2(128);
  const SpeedField s(g, std::vector<double>(g.size(), 1.0));
  const auto z = pml_damping_profile(128, 16, 1.0 / 128, 1.0);
  const PmlConfig cfg(g, s, z, z, 1.0 / 1024, 1024);  // t = 1
  const PmlState out = pml_propagate_coupling(PmlState(pulse(g)), cfg);
  double e0 = 0, e1 = 0;
  const WaveState w = pulse(g);
  for (std::size_t i = 0; i < g.size(); ++i) {
    e0 += w.u[i] * w.u[i];
    e1 += out.wave.u[i] * out.wave.u[i] + out.wave.udot[i] * out.wave.udot[i] * 1e-4;
  }
  CHECK(out.finite());
  CHECK(e1 < 1e-2 * e0);
}

TEST_CASE("errors follow PropagatorConfig") {
  const Grid g = grid2(32);
  const SpeedField s(g, std::vector<double>(g.size(), 1.0));
  const std::vector<double> z(32, 0.0);
  CHECK_THROWS_AS(PmlConfig(g, s, z, z, 1.0 / 32, 4), std::invalid_argument);                   // CFL
  CHECK_THROWS_AS(PmlConfig(g, s, std::vector<double>(31, 0.0), z, 0.001, 4), std::invalid_argument);
  CHECK_THROWS_AS(PmlConfig(g, s, std::vector<double>(32, -1.0), z, 0.001, 4), std::invalid_argument);
  const PmlConfig cfg(g, s, z, z, 0.001, 4);
  WaveState w = pulse(g);
  w.u[5] = std::numeric_limits<double>::infinity();
  CHECK_THROWS_AS(pml_propagate_coupling(PmlState(w), cfg), PropagationDiverged);
}

TEST_CASE("plain parareal with the layer: converged slices are exact") {
  const Grid fg = grid2(64), cg = grid2(16);
  const SpeedField fs(fg, std::vector<double>(fg.size(), 1.0)), cs(cg, std::vector<double>(cg.size(), 1.0));
  const auto zf = pml_damping_profile(64, 8, 1.0 / 64, 1.0), zc = pml_damping_profile(16, 2, 1.0 / 16, 1.0);
  const PmlConfig fine(fg, fs, zf, zf, 1.0 / 512, 16), coarse(cg, cs, zc, zc, 1.0 / 64, 2);
  const GridTransfer t(cg, fg, InterpKind::fourier);
  std::vector<std::vector<double>> err;
  const auto it = pml_plain_parareal(pulse(fg), fine, coarse, t, 6, 3, &err);
  REQUIRE(it.size() == 7);
  REQUIRE(err.size() == 3);
  for (int k = 0; k < 3; ++k)
    for (int n = 0; n <= k + 1; ++n) CHECK(err[size_t(k)][size_t(n)] == 0.0);
  // the first iterate's slice 1 is one fine coupling of the initial state
  const PmlState f1 = pml_propagate_coupling(PmlState(pulse(fg)), fine);
  CHECK(it[1].wave.u == f1.wave.u);
}
