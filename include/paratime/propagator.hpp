// paratime_b200 drop-in for /root/reference/proj/include/paratime/propagator.hpp:12-31.
// The Verlet stepping runs in the batched sm_100a kernels (libparatime_b200).
#pragma once

#include <cstddef>
#include <memory>
#include <span>
#include <vector>

#include "paratime/grid.hpp"

namespace paratime {

/// Propagator configuration; the constructor enforces dt*max(c)/min(h) <= 1/sqrt(d)
/// (propagator.cpp:11-27).  The device-side copy of the speed field is created on first use.
struct PropagatorConfig {
  Grid grid;
  SpeedField speed;
  double dt;
  std::size_t steps_per_coupling;

  PropagatorConfig(Grid g, SpeedField s, double dt_in, std::size_t steps);

  struct Device;                             // opaque device handle cache
  mutable std::shared_ptr<Device> device_;   // implementation detail
};

/// Periodic 5-point Laplacian (reference operation order, bitwise).
std::vector<double> laplacian(const std::vector<double>& field, const Grid& grid);

/// One velocity-Verlet step; throws PropagationDiverged on a non-finite result.
WaveState step(const WaveState& state, const PropagatorConfig& cfg);

/// steps_per_coupling Verlet steps; throws PropagationDiverged on a non-finite result.
WaveState propagate_coupling(const WaveState& state, const PropagatorConfig& cfg);

/// Batched extension: every state advanced by one coupling in one device call.
/// diverged[i] is set (and states[i] left as computed) where propagate_coupling would throw.
void propagate_coupling_batch(std::span<WaveState> states, const PropagatorConfig& cfg,
                              std::vector<bool>* diverged = nullptr);

/// Arithmetic of the device propagator: fast (FMA, <= 1e-12 of the reference) or exact
/// (the reference's operations in its order, bitwise).  Default: fast, or PTB_MODE=exact.
enum class PropagatorMode { fast, exact };
void set_propagator_mode(PropagatorMode mode);
PropagatorMode propagator_mode();

}  // namespace paratime
