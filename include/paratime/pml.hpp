// paratime_b200 extension (no counterpart in /root/reference/proj): the absorbing layer of
// BASELINE.json config 4.  The reference propagator is periodic only (propagator.hpp:12-31,
// propagator.cpp:31-105); this adds a layered propagator in the same value-type style, running in
// libparatime_b200's k_pml kernels (scheme: oracle/pml_np.py).
#pragma once

#include <cstddef>
#include <memory>
#include <span>
#include <vector>

#include "paratime/grid.hpp"

namespace paratime {

/// Wave state plus the auxiliary fields of the layer (zero wherever zeta_x = zeta_y = 0).
struct PmlState {
  WaveState wave;
  std::vector<double> px;
  std::vector<double> py;

  explicit PmlState(WaveState w);  // auxiliary fields zero
  PmlState(WaveState w, std::vector<double> px_in, std::vector<double> py_in);
  bool finite() const;
};

/// Quadratic damping profile zeta = z0 (d/L)^2 on `width` cells at both ends of an axis of n
/// cells, z0 = 1.5 cmax ln(1/reflection) / (width h).
std::vector<double> pml_damping_profile(std::size_t n, std::size_t width, double h, double cmax,
                                        double reflection = 1e-4);

/// 2D layered propagator configuration; validates like PropagatorConfig (CFL, dt, steps) plus
/// non-negative damping.  zeta_y: one value per row (axis 0), zeta_x: one per column (axis 1).
struct PmlConfig {
  Grid grid;
  SpeedField speed;
  std::vector<double> zeta_y;
  std::vector<double> zeta_x;
  double dt;
  std::size_t steps_per_coupling;

  PmlConfig(Grid g, SpeedField s, std::vector<double> zy, std::vector<double> zx, double dt_in, std::size_t steps);

  struct Device;
  mutable std::shared_ptr<Device> device_;
};

/// steps_per_coupling layered steps; throws PropagationDiverged on a non-finite result.
PmlState pml_propagate_coupling(const PmlState& state, const PmlConfig& cfg);

/// Every state advanced by one coupling in one device call; diverged[i] set where
/// pml_propagate_coupling would throw.
void pml_propagate_coupling_batch(std::span<PmlState> states, const PmlConfig& cfg,
                                  std::vector<bool>* diverged = nullptr);

/// Plain parareal (parareal.cpp:201-237, Eq. 2) on the layered state: fine and coarse layered
/// propagators on transfer's fine / coarse grids with the same coupling interval; iterate 0 is
/// the interpolated serial coarse chain.  Returns the last iterate (n_couplings + 1 states);
/// errors[k][n] (optional) = ||[u; udot] - serial fine||_2 / ||initial [u; udot]||_2.
std::vector<PmlState> pml_plain_parareal(const WaveState& init, const PmlConfig& fine, const PmlConfig& coarse,
                                         const GridTransfer& transfer, std::size_t n_couplings, int iterations,
                                         std::vector<std::vector<double>>* errors = nullptr);

}  // namespace paratime
