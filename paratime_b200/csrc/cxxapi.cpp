// C++ drop-in API (include/paratime/*.hpp) over the extern "C" device layer.
//
// Value types (Grid, WaveState, SpeedField, GridTransfer, PropagatorConfig, EnergyComponents,
// PhaseCorrector, ParaRun) live on the host exactly as in /root/reference/proj; every numerical
// operation is a call into libparatime_b200's C ABI on a process-wide context (device
// $PTB_DEVICE, default 0).  Validation messages and exception types follow the reference:
// std::invalid_argument for bad grids/shapes/CFL/tol, PropagationDiverged for a non-finite
// coupling, std::domain_error for zero reference energy/displacement.

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <cstring>
#include <sstream>
#include <filesystem>
#include <fstream>
#include <cstdio>
#include <istream>
#include <ostream>
#include <map>
#include <numeric>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>

#include "paratime/energy_map.hpp"
#include "paratime/errors.hpp"
#include "paratime/run_files.hpp"
#include "paratime/speed_model.hpp"
#include "paratime/grid.hpp"
#include "paratime/parareal.hpp"
#include "paratime/pml.hpp"
#include "paratime/procrustes.hpp"
#include "paratime/propagator.hpp"
#include "paratime_b200.h"

namespace paratime {
namespace {

std::mutex g_mu;

ptb_context* ctx() {
  static ptb_context* c = [] {
    int dev = 0;
    if (const char* e = std::getenv("PTB_DEVICE")) dev = std::atoi(e);
    ptb_context* h = nullptr;
    if (ptb_context_create(dev, &h) != PTB_OK)
      throw std::runtime_error(std::string("paratime_b200: no CUDA device: ") + ptb_last_error());
    return h;
  }();
  return c;
}

void check(ptb_status s) {
  if (s == PTB_OK) return;
  const std::string msg = ptb_last_error();
  switch (s) {
    case PTB_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case PTB_DIVERGED: throw PropagationDiverged(msg);
    case PTB_DOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error(msg);
  }
}

ptb_grid cgrid(const Grid& g) {
  ptb_grid o{};
  o.dim = g.dim();
  o.n[0] = g.points(0);
  o.h[0] = g.spacing(0);
  o.n[1] = g.dim() == 2 ? g.points(1) : 1;
  o.h[1] = g.dim() == 2 ? g.spacing(1) : 1.0;
  return o;
}

// device buffer of doubles on the default context
struct DBuf {
  double* p = nullptr;
  size_t n = 0;
  explicit DBuf(size_t count) : n(count) {
    void* v = nullptr;
    check(ptb_device_alloc(ctx(), std::max<size_t>(1, n) * sizeof(double), &v));
    p = static_cast<double*>(v);
  }
  DBuf(const std::vector<double>& host) : DBuf(host.size()) { up(host.data(), host.size()); }
  ~DBuf() { ptb_device_free(ctx(), p); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  void up(const double* h, size_t count, size_t off = 0) {
    if (count) check(ptb_memcpy_h2d(ctx(), p + off, h, count * sizeof(double)));
  }
  std::vector<double> down(size_t count, size_t off = 0) const {
    std::vector<double> h(count);
    if (count) check(ptb_memcpy_d2h(ctx(), h.data(), p + off, count * sizeof(double)));
    return h;
  }
};

void check_same_grid(const Grid& a, const Grid& b, const char* what) {
  if (a != b) throw std::invalid_argument(std::string(what) + ": grid mismatch");
}

bool all_finite(const std::vector<double>& v) {
  return std::all_of(v.begin(), v.end(), [](double x) { return std::isfinite(x); });
}

PropagatorMode& mode_ref() {
  static PropagatorMode m = [] {
    const char* e = std::getenv("PTB_MODE");
    return (e && std::string(e) == "exact") ? PropagatorMode::exact : PropagatorMode::fast;
  }();
  return m;
}

int mode_id() { return mode_ref() == PropagatorMode::exact ? PTB_MODE_EXACT : PTB_MODE_FAST; }

size_t fingerprint(const Grid& g, const std::vector<double>& c, double dt, size_t steps) {
  size_t h = std::hash<double>()(dt) ^ (steps * 0x9e3779b97f4a7c15ULL);
  for (int a = 0; a < g.dim(); ++a) h = h * 31 + std::hash<double>()(g.spacing(a)) + g.points(a);
  for (double v : c) h = h * 1099511628211ULL + std::hash<double>()(v);
  return h;
}

// transfer handles are cached per (coarse, fine, kind)
ptb_transfer* transfer_of(const GridTransfer& t) {
  using Key = std::tuple<int, size_t, size_t, double, double, size_t, size_t, double, double, int>;
  static std::map<Key, ptb_transfer*> cache;
  const ptb_grid c = cgrid(t.coarse), f = cgrid(t.fine);
  const Key key{c.dim, c.n[0], c.n[1], c.h[0], c.h[1], f.n[0], f.n[1], f.h[0], f.h[1], int(t.kind)};
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  ptb_transfer* h = nullptr;
  check(ptb_transfer_create(ctx(), &c, &f, t.kind == InterpKind::fourier ? PTB_INTERP_FOURIER : PTB_INTERP_LINEAR, &h));
  cache.emplace(key, h);
  return h;
}

int scheme_id(GradientScheme s) { return static_cast<int>(s); }

}  // namespace

// ------------------------------------------------------------------------ grid.hpp
//
// Host value types.  The checks and their messages are the reference's contract (grid.cpp:13-119):
// the same std::invalid_argument text is what CHECK_THROWS_AS cases and callers see.

namespace {
void require(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}
bool positive_finite(double v) { return v > 0.0 && std::isfinite(v); }

// elementwise a (op) b on both fields of a state; grids must agree
template <typename Op>
WaveState combine(const WaveState& a, const WaveState& b, const char* what, Op op) {
  check_same_grid(a.grid, b.grid, what);
  WaveState o = a;
  std::transform(o.u.begin(), o.u.end(), b.u.begin(), o.u.begin(), op);
  std::transform(o.udot.begin(), o.udot.end(), b.udot.begin(), o.udot.begin(), op);
  return o;
}
}  // namespace

Grid::Grid(std::vector<std::size_t> points_per_axis, std::vector<double> spacing)
    : n_(std::move(points_per_axis)), h_(std::move(spacing)) {
  require(!n_.empty() && n_.size() <= 2 && n_.size() == h_.size(), "Grid: dimension must be 1 or 2 with matching spacing");
  for (std::size_t a = 0; a < n_.size(); ++a) {  // axis by axis: the first bad axis names the error
    require(n_[a] >= 4, "Grid: need at least 4 points per axis");
    require(positive_finite(h_[a]), "Grid: spacing must be positive");
  }
}

std::size_t Grid::size() const {
  return std::accumulate(n_.begin(), n_.end(), std::size_t(1), std::multiplies<std::size_t>());
}

double Grid::cell_volume() const { return std::accumulate(h_.begin(), h_.end(), 1.0, std::multiplies<double>()); }

bool Grid::operator==(const Grid& o) const { return n_ == o.n_ && h_ == o.h_; }

WaveState::WaveState(Grid g, std::vector<double> u_in, std::vector<double> udot_in)
    : grid(std::move(g)), u(std::move(u_in)), udot(std::move(udot_in)) {
  require(u.size() == grid.size() && udot.size() == grid.size(), "WaveState: field size does not match grid");
}

WaveState::WaveState(Grid g) : grid(std::move(g)), u(grid.size(), 0.0), udot(grid.size(), 0.0) {}

bool WaveState::finite() const { return all_finite(u) && all_finite(udot); }

WaveState operator+(const WaveState& a, const WaveState& b) { return combine(a, b, "state add", std::plus<double>()); }

WaveState operator-(const WaveState& a, const WaveState& b) {
  return combine(a, b, "state subtract", std::minus<double>());
}

WaveState operator*(double s, const WaveState& a) {
  WaveState o = a;
  for (auto* f : {&o.u, &o.udot})
    for (double& x : *f) x *= s;
  return o;
}

SpeedField::SpeedField(Grid g, std::vector<double> c_in) : grid(std::move(g)), c(std::move(c_in)) {
  require(c.size() == grid.size(), "SpeedField: field size does not match grid");
  require(std::all_of(c.begin(), c.end(), positive_finite), "SpeedField: wave speed must be strictly positive and finite");
}

GridTransfer::GridTransfer(Grid coarse_in, Grid fine_in, InterpKind kind_in)
    : coarse(std::move(coarse_in)), fine(std::move(fine_in)), kind(kind_in) {
  require(coarse.dim() == fine.dim(), "GridTransfer: dimension mismatch");
  for (int a = 0; a < coarse.dim(); ++a) {
    const std::size_t nc = coarse.points(a), nf = fine.points(a);
    require(nf % nc == 0, "GridTransfer: fine points must be an integer multiple of coarse points");
    ratio.push_back(nf / nc);
    const double ec = coarse.extent(a), ef = fine.extent(a);
    require(std::abs(ec - ef) <= 1e-12 * std::max(ec, ef), "GridTransfer: coarse and fine extents differ; grids are not nested");
  }
}

bool GridTransfer::identity() const {
  return std::all_of(ratio.begin(), ratio.end(), [](size_t r) { return r == 1; });
}

std::vector<double> restrict_field(const std::vector<double>& fine_field, const GridTransfer& t) {
  if (fine_field.size() != t.fine.size())
    throw std::invalid_argument("restrict_field: input does not live on the fine grid");
  DBuf in(fine_field), out(t.coarse.size());
  check(ptb_restrict_batch(transfer_of(t), 1, in.p, out.p));
  return out.down(t.coarse.size());
}

WaveState restrict_state(const WaveState& s, const GridTransfer& t) {
  if (s.grid != t.fine) throw std::invalid_argument("restrict_state: state does not live on the fine grid");
  return WaveState(t.coarse, restrict_field(s.u, t), restrict_field(s.udot, t));
}

std::vector<double> interpolate_field(const std::vector<double>& coarse_field, const GridTransfer& t) {
  if (coarse_field.size() != t.coarse.size())
    throw std::invalid_argument("interpolate_field: input does not live on the coarse grid");
  DBuf in(coarse_field), out(t.fine.size());
  check(ptb_interpolate_batch(transfer_of(t), 1, in.p, out.p));
  return out.down(t.fine.size());
}

WaveState interpolate_state(const WaveState& s, const GridTransfer& t) {
  if (s.grid != t.coarse) throw std::invalid_argument("interpolate_state: state does not live on the coarse grid");
  return WaveState(t.fine, interpolate_field(s.u, t), interpolate_field(s.udot, t));
}

SpeedField resize_speed(const SpeedField& fine_speed, const Grid& coarse) {
  const GridTransfer t(coarse, fine_speed.grid, InterpKind::linear);
  return SpeedField(coarse, restrict_field(fine_speed.c, t));
}

// ------------------------------------------------------------------ propagator.hpp

struct PropagatorConfig::Device {
  ptb_propagator* p = nullptr;
  size_t hash = 0;
  ~Device() { ptb_propagator_destroy(p); }
};

PropagatorConfig::PropagatorConfig(Grid g, SpeedField s, double dt_in, std::size_t steps)
    : grid(std::move(g)), speed(std::move(s)), dt(dt_in), steps_per_coupling(steps) {
  if (speed.grid != grid) throw std::invalid_argument("PropagatorConfig: speed field lives on a different grid");
  if (!(dt > 0.0) || !std::isfinite(dt)) throw std::invalid_argument("PropagatorConfig: dt must be positive");
  if (steps_per_coupling == 0) throw std::invalid_argument("PropagatorConfig: steps_per_coupling must be positive");
  const double cmax = *std::max_element(speed.c.begin(), speed.c.end());
  double hmin = grid.spacing(0);
  for (int a = 1; a < grid.dim(); ++a) hmin = std::min(hmin, grid.spacing(a));
  const double cfl = dt * cmax / hmin, bound = 1.0 / std::sqrt(double(grid.dim()));
  if (cfl > bound * (1.0 + 1e-12))
    throw std::invalid_argument("PropagatorConfig: CFL violated, dt*max(c)/min(h) = " + std::to_string(cfl) + " > " +
                                std::to_string(bound));
}

static ptb_propagator* device_of(const PropagatorConfig& cfg) {
  const size_t h = fingerprint(cfg.grid, cfg.speed.c, cfg.dt, cfg.steps_per_coupling);
  std::lock_guard<std::mutex> lock(g_mu);
  if (!cfg.device_ || cfg.device_->hash != h) {
    auto d = std::make_shared<PropagatorConfig::Device>();
    const ptb_grid g = cgrid(cfg.grid);
    check(ptb_propagator_create(ctx(), &g, cfg.speed.c.data(), cfg.dt, cfg.steps_per_coupling, &d->p));
    d->hash = h;
    cfg.device_ = d;
  }
  return cfg.device_->p;
}

void set_propagator_mode(PropagatorMode m) { mode_ref() = m; }
PropagatorMode propagator_mode() { return mode_ref(); }

std::vector<double> laplacian(const std::vector<double>& field, const Grid& grid) {
  if (field.size() != grid.size()) throw std::invalid_argument("laplacian: field size does not match grid");
  DBuf in(field), out(field.size());
  const ptb_grid g = cgrid(grid);
  check(ptb_laplacian_batch(ctx(), &g, 1, in.p, out.p));
  return out.down(field.size());
}

WaveState step(const WaveState& state, const PropagatorConfig& cfg) {
  if (state.grid != cfg.grid) throw std::invalid_argument("step: state does not live on the propagator grid");
  const size_t n = state.u.size();
  DBuf u(state.u), v(state.udot);
  check(ptb_propagate_steps_batch(device_of(cfg), 1, 1, u.p, v.p, nullptr, mode_id()));
  WaveState out(state.grid, u.down(n), v.down(n));
  if (!out.finite()) throw PropagationDiverged("step: non-finite state produced");
  return out;
}

WaveState propagate_coupling(const WaveState& state, const PropagatorConfig& cfg) {
  if (state.grid != cfg.grid)
    throw std::invalid_argument("propagate_coupling: state does not live on the propagator grid");
  WaveState out(state.grid);
  check(ptb_propagate_coupling_host(device_of(cfg), state.u.data(), state.udot.data(), out.u.data(), out.udot.data(),
                                    mode_id()));
  return out;
}

void propagate_coupling_batch(std::span<WaveState> states, const PropagatorConfig& cfg, std::vector<bool>* diverged) {
  const size_t B = states.size(), n = cfg.grid.size();
  for (const auto& s : states)
    if (s.grid != cfg.grid) throw std::invalid_argument("propagate_coupling_batch: state not on the propagator grid");
  std::vector<double> u(B * n), v(B * n);
  for (size_t b = 0; b < B; ++b) {
    std::copy(states[b].u.begin(), states[b].u.end(), u.begin() + long(b * n));
    std::copy(states[b].udot.begin(), states[b].udot.end(), v.begin() + long(b * n));
  }
  std::vector<int32_t> flags(B, 0);
  check(ptb_propagate_batch_host(device_of(cfg), B, u.data(), v.data(), u.data(), v.data(), flags.data(), mode_id()));
  for (size_t b = 0; b < B; ++b) {
    std::copy(u.begin() + long(b * n), u.begin() + long((b + 1) * n), states[b].u.begin());
    std::copy(v.begin() + long(b * n), v.begin() + long((b + 1) * n), states[b].udot.begin());
  }
  if (diverged) {
    diverged->assign(B, false);
    for (size_t b = 0; b < B; ++b) (*diverged)[b] = flags[b] != 0;
  }
}

// ------------------------------------------------------------------ energy_map.hpp

GradientScheme gradient_scheme_from_string(const std::string& name) {
  if (name == "fd2") return GradientScheme::fd2;
  if (name == "fd4") return GradientScheme::fd4;
  if (name == "fd6") return GradientScheme::fd6;
  if (name == "fd8") return GradientScheme::fd8;
  if (name == "spectral") return GradientScheme::spectral;
  throw std::invalid_argument("unknown gradient scheme: " + name);
}

std::string to_string(GradientScheme s) {
  switch (s) {
    case GradientScheme::fd2: return "fd2";
    case GradientScheme::fd4: return "fd4";
    case GradientScheme::fd6: return "fd6";
    case GradientScheme::fd8: return "fd8";
    case GradientScheme::spectral: return "spectral";
  }
  return "?";
}

const std::vector<double>& stencil_coefficients(GradientScheme s) {
  static const std::vector<double> t2{1.0 / 2.0}, t4{2.0 / 3.0, -1.0 / 12.0}, t6{3.0 / 4.0, -3.0 / 20.0, 1.0 / 60.0},
      t8{4.0 / 5.0, -1.0 / 5.0, 4.0 / 105.0, -1.0 / 280.0};
  switch (s) {
    case GradientScheme::fd2: return t2;
    case GradientScheme::fd4: return t4;
    case GradientScheme::fd6: return t6;
    case GradientScheme::fd8: return t8;
    case GradientScheme::spectral: break;
  }
  throw std::invalid_argument("stencil_coefficients: spectral scheme has no stencil");
}

EnergyComponents to_energy_components(const WaveState& state, const SpeedField& speed, GradientScheme scheme) {
  if (state.grid != speed.grid) throw std::invalid_argument("to_energy_components: state/speed grid mismatch");
  const Grid& g = state.grid;
  const size_t n = g.size(), d = size_t(g.dim());
  DBuf u(state.u), v(state.udot), c(speed.c), out((d + 1) * n), mean(1);
  const ptb_grid cg = cgrid(g);
  check(ptb_energy_components_batch(ctx(), &cg, c.p, scheme_id(scheme), 1, u.p, v.p, out.p, (d + 1) * n, mean.p));
  const std::vector<double> st = out.down((d + 1) * n);
  EnergyComponents comp{g, {}, std::vector<double>(st.begin() + long(d * n), st.end()), mean.down(1)[0]};
  for (size_t a = 0; a < d; ++a) comp.grad.emplace_back(st.begin() + long(a * n), st.begin() + long((a + 1) * n));
  return comp;
}

std::vector<double> gradient_axis(const std::vector<double>& field, const Grid& grid, int axis, GradientScheme scheme) {
  if (field.size() != grid.size()) throw std::invalid_argument("gradient_axis: field size does not match grid");
  if (axis < 0 || axis >= grid.dim()) throw std::invalid_argument("gradient_axis: axis out of range");
  const WaveState s(grid, field, std::vector<double>(grid.size(), 0.0));
  return to_energy_components(s, SpeedField(grid, std::vector<double>(grid.size(), 1.0)), scheme)
      .grad[size_t(axis)];
}

WaveState from_energy_components(const EnergyComponents& comp, const SpeedField& speed) {
  const Grid& g = comp.grid;
  if (g != speed.grid) throw std::invalid_argument("from_energy_components: grid mismatch");
  if (int(comp.grad.size()) != g.dim())
    throw std::invalid_argument("from_energy_components: wrong number of gradient blocks");
  const std::vector<double> st = stack_components(comp);
  DBuf s(st), mean(std::vector<double>{comp.mean_u}), c(speed.c), u(g.size()), v(g.size());
  const ptb_grid cg = cgrid(g);
  check(ptb_from_energy_components_batch(ctx(), &cg, c.p, 1, s.p, st.size(), mean.p, u.p, v.p));
  return WaveState(g, u.down(g.size()), v.down(g.size()));
}

double energy(const EnergyComponents& comp) {
  double acc = 0.0;
  for (const auto& b : comp.grad)
    for (double x : b) acc += x * x;
  for (double x : comp.momentum) acc += x * x;
  return 0.5 * acc * comp.grid.cell_volume();
}

namespace {
// {|Lambda(a-b)|^2, |Lambda(b)|^2, |ua-ub|^2, |ub|^2} on the device
std::vector<double> pair_sums(const WaveState& a, const WaveState& b, const SpeedField& speed, GradientScheme scheme) {
  DBuf ua(a.u), va(a.udot), ub(b.u), vb(b.udot), c(speed.c), out(4);
  const ptb_grid g = cgrid(a.grid);
  check(ptb_energy_sums_batch(ctx(), &g, c.p, scheme_id(scheme), 1, ua.p, va.p, ub.p, vb.p, out.p));
  return out.down(4);
}
}  // namespace

double energy(const WaveState& state, const SpeedField& speed, GradientScheme scheme) {
  const WaveState zero(state.grid);
  return 0.5 * pair_sums(state, zero, speed, scheme)[0] * state.grid.cell_volume();
}

double energy_error(const WaveState& a, const WaveState& b, const SpeedField& speed, GradientScheme scheme) {
  if (a.grid != b.grid) throw std::invalid_argument("energy_error: states live on different grids");
  const std::vector<double> s = pair_sums(a, b, speed, scheme);
  const double vol = a.grid.cell_volume();
  const double ref = 0.5 * s[1] * vol;
  if (ref == 0.0) throw std::domain_error("energy_error: reference state has zero energy");
  return std::sqrt((0.5 * s[0] * vol) / ref);
}

double l2_error(const WaveState& a, const WaveState& b) {
  if (a.grid != b.grid) throw std::invalid_argument("l2_error: states live on different grids");
  const std::vector<double> s =
      pair_sums(a, b, SpeedField(a.grid, std::vector<double>(a.grid.size(), 1.0)), GradientScheme::fd2);
  if (s[3] == 0.0) throw std::domain_error("l2_error: reference displacement is zero");
  return std::sqrt(s[2] / s[3]);
}

// ------------------------------------------------------------------ procrustes.hpp

double Matrix::squaredNorm() const {
  double acc = 0.0;
  for (double v : data_) acc += v * v;
  return acc;
}

double Matrix::norm() const { return std::sqrt(squaredNorm()); }

Matrix operator-(const Matrix& a, const Matrix& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) throw std::invalid_argument("Matrix: shape mismatch");
  Matrix o(a.rows(), a.cols());
  for (Index k = 0; k < a.rows() * a.cols(); ++k) o.data()[k] = a.data()[k] - b.data()[k];
  return o;
}

Matrix operator+(const Matrix& a, const Matrix& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) throw std::invalid_argument("Matrix: shape mismatch");
  Matrix o(a.rows(), a.cols());
  for (Index k = 0; k < a.rows() * a.cols(); ++k) o.data()[k] = a.data()[k] + b.data()[k];
  return o;
}

PhaseCorrector::PhaseCorrector(Matrix left, std::vector<double> sv, Matrix right, double tol)
    : left_(std::move(left)), sv_(std::move(sv)), right_(std::move(right)), tol_(tol) {
  if (left_.rows() != right_.rows() || left_.cols() != right_.cols() || left_.cols() != Index(sv_.size()))
    throw std::invalid_argument("PhaseCorrector: inconsistent factor shapes");
}

namespace {
struct DevCorr {
  ptb_corrector* h = nullptr;
  DevCorr() { check(ptb_corrector_create(ctx(), &h)); }
  explicit DevCorr(const PhaseCorrector& c) : DevCorr() {
    if (!c.empty())
      check(ptb_corrector_set(h, size_t(c.rows()), size_t(c.rank()), c.left().data(), c.singular_values().data(),
                              c.right().data(), c.tol()));
  }
  ~DevCorr() { ptb_corrector_destroy(h); }
  PhaseCorrector download(double tol) const {
    size_t rows = 0, rank = 0;
    check(ptb_corrector_shape(h, &rows, &rank));
    Matrix X{Index(rows), Index(rank)}, Y{Index(rows), Index(rank)};
    std::vector<double> S(rank);
    check(ptb_corrector_factors(h, X.data(), S.data(), Y.data()));
    return PhaseCorrector(std::move(X), std::move(S), std::move(Y), tol);
  }
};

void check_tol(double tol) {
  if (!(tol > 0.0) || !(tol < 1.0)) throw std::invalid_argument("truncation tolerance must lie in (0, 1)");
}
}  // namespace

std::vector<double> PhaseCorrector::apply(const std::vector<double>& stacked) const {
  if (Index(stacked.size()) != rows())
    throw std::invalid_argument("PhaseCorrector: stacked length does not match rows");
  if (rank() == 0) return std::vector<double>(stacked.size(), 0.0);
  DevCorr d(*this);
  DBuf in(stacked), out(stacked.size());
  check(ptb_corrector_apply_batch(d.h, 1, in.p, out.p));
  return out.down(stacked.size());
}

PhaseCorrector PhaseCorrector::drop_leading(Index count) const {
  if (count < 0) throw std::invalid_argument("drop_leading: negative count");
  const Index keep = std::max<Index>(0, rank() - count), first = rank() - keep;
  Matrix l(rows(), keep), r(rows(), keep);
  std::copy(left_.col(first), left_.col(first) + rows() * keep, l.data());
  std::copy(right_.col(first), right_.col(first) + rows() * keep, r.data());
  return PhaseCorrector(std::move(l), std::vector<double>(sv_.begin() + first, sv_.end()), std::move(r), tol_);
}

std::vector<double> stack_components(const EnergyComponents& comp) {
  std::vector<double> out;
  out.reserve((comp.grad.size() + 1) * comp.grid.size());
  for (const auto& b : comp.grad) out.insert(out.end(), b.begin(), b.end());
  out.insert(out.end(), comp.momentum.begin(), comp.momentum.end());
  return out;
}

EnergyComponents unstack_components(const std::vector<double>& stacked, const Grid& grid, double mean_u) {
  const size_t n = grid.size(), d = size_t(grid.dim());
  if (stacked.size() != (d + 1) * n) throw std::invalid_argument("unstack_components: length does not match grid");
  EnergyComponents comp{grid, {}, std::vector<double>(stacked.begin() + long(d * n), stacked.end()), mean_u};
  for (size_t a = 0; a < d; ++a) comp.grad.emplace_back(stacked.begin() + long(a * n), stacked.begin() + long((a + 1) * n));
  return comp;
}

std::pair<SnapshotMatrix, SnapshotMatrix> assemble_snapshots(std::span<const WaveState> fine_states,
                                                             std::span<const WaveState> coarse_states,
                                                             const GridTransfer& transfer,
                                                             const SpeedField& coarse_speed, GradientScheme scheme) {
  if (fine_states.empty() || fine_states.size() != coarse_states.size())
    throw std::invalid_argument("assemble_snapshots: need equal, nonempty snapshot lists");
  const Index rows = Index((transfer.coarse.dim() + 1) * transfer.coarse.size());
  const Index cols = Index(fine_states.size());
  SnapshotMatrix F(rows, cols), G(rows, cols);
  for (Index k = 0; k < cols; ++k) {
    const auto f = stack_components(
        to_energy_components(restrict_state(fine_states[size_t(k)], transfer), coarse_speed, scheme));
    const auto g = stack_components(to_energy_components(coarse_states[size_t(k)], coarse_speed, scheme));
    std::copy(f.begin(), f.end(), F.col(k));
    std::copy(g.begin(), g.end(), G.col(k));
  }
  return {std::move(F), std::move(G)};
}

PhaseCorrector procrustes_solve(const SnapshotMatrix& F, const SnapshotMatrix& G, double tol) {
  check_tol(tol);
  if (F.rows() != G.rows() || F.cols() != G.cols())
    throw std::invalid_argument("procrustes_solve: F and G must have the same shape");
  if (F.cols() > F.rows()) throw std::invalid_argument("procrustes_solve: more snapshots than rows");
  if (F.cols() == 0) throw std::invalid_argument("procrustes_solve: empty data");
  DevCorr d;
  DBuf f(size_t(F.rows() * F.cols())), g(size_t(G.rows() * G.cols()));
  f.up(F.data(), f.n);
  g.up(G.data(), g.n);
  check(ptb_procrustes_solve(d.h, size_t(F.rows()), size_t(F.cols()), f.p, g.p, tol));
  return d.download(tol);
}

PhaseCorrector update_svd(const PhaseCorrector& corrector, const SnapshotMatrix& F, const SnapshotMatrix& G, double tol) {
  check_tol(tol);
  if (F.rows() != G.rows() || F.cols() != G.cols())
    throw std::invalid_argument("update_svd: F and G must have the same shape");
  if (!corrector.empty() && F.rows() != corrector.rows())
    throw std::invalid_argument("update_svd: block rows do not match corrector");
  DevCorr d(corrector);
  DBuf f(size_t(F.rows() * F.cols())), g(size_t(G.rows() * G.cols()));
  f.up(F.data(), f.n);
  g.up(G.data(), g.n);
  check(ptb_corrector_update(d.h, size_t(F.rows()), size_t(F.cols()), f.p, g.p, tol));
  return d.download(tol);
}

EnergyComponents apply_corrector(const PhaseCorrector& corrector, const EnergyComponents& comp) {
  return unstack_components(corrector.apply(stack_components(comp)), comp.grid, comp.mean_u);
}

double relative_residual(const PhaseCorrector& corrector, const SnapshotMatrix& F, const SnapshotMatrix& G) {
  const double fnorm = F.norm();
  if (fnorm == 0.0) return 0.0;
  if (corrector.rank() == 0) return 1.0;
  DevCorr d(corrector);
  DBuf f(size_t(F.rows() * F.cols())), g(size_t(G.rows() * G.cols()));
  f.up(F.data(), f.n);
  g.up(G.data(), g.n);
  double r = 0.0;
  check(ptb_relative_residual(d.h, size_t(F.rows()), size_t(F.cols()), f.p, g.p, &r));
  return r;
}

// ------------------------------------------------------------------ parareal.hpp

CouplingSchedule::CouplingSchedule(double T_in, double dt_com_in, std::size_t n, PropagatorConfig fine,
                                   PropagatorConfig coarse)
    : T(T_in), dt_com(dt_com_in), n_couplings(n), fine_cfg(std::move(fine)), coarse_cfg(std::move(coarse)) {
  // parareal.cpp:172-188: N dt_com = T to 1e-9, m dt = dt_com to 1e-12 for both propagators
  require(T > 0.0 && dt_com > 0.0 && n_couplings > 0, "CouplingSchedule: T, dt_com, N must be positive");
  require(std::abs(double(n_couplings) * dt_com - T) <= 1e-9 * T, "CouplingSchedule: N * dt_com must equal T");
  const auto spans = [this](const PropagatorConfig& c) {
    return std::abs(double(c.steps_per_coupling) * c.dt - dt_com) <= 1e-12 * dt_com;
  };
  require(spans(fine_cfg), "CouplingSchedule: fine steps_per_coupling * dt != dt_com");
  require(spans(coarse_cfg), "CouplingSchedule: coarse steps_per_coupling * dt != dt_com");
}

std::vector<WaveState> serial_fine(const WaveState& init, const CouplingSchedule& schedule) {
  if (init.grid != schedule.fine_cfg.grid)
    throw std::invalid_argument("serial_fine: initial state must live on the fine grid");
  std::vector<WaveState> states{init};
  states.reserve(schedule.n_couplings + 1);
  for (size_t n = 1; n <= schedule.n_couplings; ++n) states.push_back(propagate_coupling(states[n - 1], schedule.fine_cfg));
  return states;
}

namespace {

ParaRun run_device(const WaveState& init, const CouplingSchedule& sch, const GridTransfer& tr, int iterations,
                   int variant, GradientScheme scheme, double tol, int remove_leading, const DriverOptions& drv) {
  if (init.grid != sch.fine_cfg.grid) throw std::invalid_argument("parareal: initial state must live on the fine grid");
  if (tr.fine != sch.fine_cfg.grid || tr.coarse != sch.coarse_cfg.grid)
    throw std::invalid_argument("parareal: transfer does not couple the schedule grids");
  if (iterations < 0) throw std::invalid_argument("parareal: negative iteration count");
  ptb_run_spec s{};
  const ptb_grid fg = cgrid(sch.fine_cfg.grid), cg = cgrid(sch.coarse_cfg.grid);
  s.dim = fg.dim;
  for (int a = 0; a < 2; ++a) {
    s.fine_n[a] = fg.n[a];
    s.fine_h[a] = fg.h[a];
    s.coarse_n[a] = cg.n[a];
    s.coarse_h[a] = cg.h[a];
  }
  s.dt_fine = sch.fine_cfg.dt;
  s.m_fine = sch.fine_cfg.steps_per_coupling;
  s.dt_coarse = sch.coarse_cfg.dt;
  s.m_coarse = sch.coarse_cfg.steps_per_coupling;
  s.T = sch.T;
  s.dt_com = sch.dt_com;
  s.n_couplings = sch.n_couplings;
  s.interp = tr.kind == InterpKind::fourier ? PTB_INTERP_FOURIER : PTB_INTERP_LINEAR;
  s.iterations = iterations;
  s.variant = variant;
  s.scheme = scheme_id(scheme);
  s.metric_scheme = scheme_id(drv.metric_scheme);
  s.tol = tol;
  s.remove_leading = remove_leading;
  s.mode = mode_id();
  const size_t N = sch.n_couplings, K = size_t(iterations), nf = init.grid.size();
  std::vector<double> ee((K + 1) * (N + 1)), l2((K + 1) * (N + 1)), res(K + 1), states, ref(2 * (N + 1) * nf);
  std::vector<int> rank(K + 1), div(K + 1);
  if (drv.keep_states) states.resize((K + 1) * (N + 1) * 2 * nf);
  check(ptb_parareal_run(ctx(), &s, sch.fine_cfg.speed.c.data(), sch.coarse_cfg.speed.c.data(), init.u.data(),
                         init.udot.data(), ee.data(), l2.data(), res.data(), rank.data(), div.data(),
                         drv.keep_states ? states.data() : nullptr, ref.data(), nullptr));
  auto state_at = [&](const std::vector<double>& buf, size_t off) {
    return WaveState(init.grid, std::vector<double>(buf.begin() + long(off), buf.begin() + long(off + nf)),
                     std::vector<double>(buf.begin() + long(off + nf), buf.begin() + long(off + 2 * nf)));
  };
  ParaRun run;
  for (size_t n = 0; n <= N; ++n) run.reference.push_back(state_at(ref, 2 * n * nf));
  for (size_t k = 0; k <= K; ++k) {
    IterationRecord rec;
    rec.energy_err.assign(ee.begin() + long(k * (N + 1)), ee.begin() + long((k + 1) * (N + 1)));
    rec.l2_err.assign(l2.begin() + long(k * (N + 1)), l2.begin() + long((k + 1) * (N + 1)));
    rec.residual = res[k];
    rec.rank = rank[k];
    rec.diverged = div[k] != 0;
    if (drv.keep_states)
      for (size_t n = 0; n <= N; ++n) rec.states.push_back(state_at(states, ((k * (N + 1) + n) * 2) * nf));
    run.iterations.push_back(std::move(rec));
  }
  return run;
}

}  // namespace

ParaRun plain_parareal(const WaveState& init, const CouplingSchedule& schedule, const GridTransfer& transfer,
                       int iterations, const DriverOptions& options) {
  return run_device(init, schedule, transfer, iterations, PTB_PLAIN, GradientScheme::fd2, 0.5, 0, options);
}

ParaRun theta_parareal(const WaveState& init, const CouplingSchedule& schedule, const GridTransfer& transfer,
                       int iterations, const ThetaOptions& o) {
  const int variant = o.omega_identity ? PTB_OMEGA_IDENTITY : (o.additive_correction ? PTB_THETA : PTB_CORRECTED_COARSE_ONLY);
  return run_device(init, schedule, transfer, iterations, variant, o.scheme, o.tol, o.remove_leading, o.driver);
}

ParaRun corrected_coarse_only(const WaveState& init, const CouplingSchedule& schedule, const GridTransfer& transfer,
                              int iterations, ThetaOptions options) {
  options.additive_correction = false;
  return theta_parareal(init, schedule, transfer, iterations, options);
}

}  // namespace paratime

// ------------------------------------------------------------------ absorbing layer (pml.hpp)
namespace paratime {

PmlState::PmlState(WaveState w) : wave(std::move(w)), px(wave.grid.size(), 0.0), py(wave.grid.size(), 0.0) {}

PmlState::PmlState(WaveState w, std::vector<double> px_in, std::vector<double> py_in)
    : wave(std::move(w)), px(std::move(px_in)), py(std::move(py_in)) {
  if (px.size() != wave.grid.size() || py.size() != wave.grid.size())
    throw std::invalid_argument("PmlState: auxiliary field size does not match grid");
}

bool PmlState::finite() const { return wave.finite() && all_finite(px) && all_finite(py); }

std::vector<double> pml_damping_profile(std::size_t n, std::size_t width, double h, double cmax, double reflection) {
  std::vector<double> z(n);
  check(ptb_pml_damping_profile(n, width, h, cmax, reflection, z.data()));
  return z;
}

struct PmlConfig::Device {
  ptb_pml* h = nullptr;
  ~Device() {
    if (h) ptb_pml_destroy(h);
  }
};

PmlConfig::PmlConfig(Grid g, SpeedField s, std::vector<double> zy, std::vector<double> zx, double dt_in,
                     std::size_t steps)
    : grid(std::move(g)), speed(std::move(s)), zeta_y(std::move(zy)), zeta_x(std::move(zx)), dt(dt_in),
      steps_per_coupling(steps) {
  check_same_grid(grid, speed.grid, "PmlConfig");
  if (grid.dim() != 2) throw std::invalid_argument("PmlConfig: the absorbing layer is two-dimensional");
  if (zeta_y.size() != grid.points(0) || zeta_x.size() != grid.points(1))
    throw std::invalid_argument("PmlConfig: one damping value per row and per column");
  auto d = std::make_shared<Device>();
  const ptb_grid cg = cgrid(grid);
  check(ptb_pml_create(ctx(), &cg, speed.c.data(), zeta_y.data(), zeta_x.data(), dt, steps_per_coupling, &d->h));
  device_ = std::move(d);
}

void pml_propagate_coupling_batch(std::span<PmlState> states, const PmlConfig& cfg, std::vector<bool>* diverged) {
  const size_t n = cfg.grid.size(), b = states.size();
  if (diverged) diverged->assign(b, false);
  if (b == 0) return;
  for (const PmlState& s : states) {
    check_same_grid(s.wave.grid, cfg.grid, "pml_propagate_coupling");
    if (s.px.size() != n || s.py.size() != n) throw std::invalid_argument("PmlState: auxiliary field size");
  }
  DBuf f(4 * b * n);
  for (size_t i = 0; i < b; ++i) {
    f.up(states[i].wave.u.data(), n, (0 * b + i) * n);
    f.up(states[i].wave.udot.data(), n, (1 * b + i) * n);
    f.up(states[i].px.data(), n, (2 * b + i) * n);
    f.up(states[i].py.data(), n, (3 * b + i) * n);
  }
  void* fl = nullptr;
  check(ptb_device_alloc(ctx(), b * sizeof(int32_t), &fl));
  std::unique_ptr<void, std::function<void(void*)>> guard(fl, [](void* q) { ptb_device_free(ctx(), q); });
  std::vector<int32_t> zeros(b, 0), flags(b, 0);
  check(ptb_memcpy_h2d(ctx(), fl, zeros.data(), b * sizeof(int32_t)));
  check(ptb_pml_propagate_batch(cfg.device_->h, 0, b, f.p, f.p + b * n, f.p + 2 * b * n, f.p + 3 * b * n,
                                static_cast<int32_t*>(fl)));
  check(ptb_memcpy_d2h(ctx(), flags.data(), fl, b * sizeof(int32_t)));
  for (size_t i = 0; i < b; ++i) {
    states[i].wave.u = f.down(n, (0 * b + i) * n);
    states[i].wave.udot = f.down(n, (1 * b + i) * n);
    states[i].px = f.down(n, (2 * b + i) * n);
    states[i].py = f.down(n, (3 * b + i) * n);
    if (diverged) (*diverged)[i] = flags[i] != 0;
  }
}

PmlState pml_propagate_coupling(const PmlState& state, const PmlConfig& cfg) {
  PmlState out = state;
  std::vector<bool> div;
  pml_propagate_coupling_batch(std::span<PmlState>(&out, 1), cfg, &div);
  if (div[0]) throw PropagationDiverged("pml_propagate_coupling: non-finite state after coupling");
  return out;
}

std::vector<PmlState> pml_plain_parareal(const WaveState& init, const PmlConfig& fine, const PmlConfig& coarse,
                                         const GridTransfer& transfer, std::size_t n_couplings, int iterations,
                                         std::vector<std::vector<double>>* errors) {
  check_same_grid(init.grid, fine.grid, "pml_plain_parareal");
  check_same_grid(transfer.fine, fine.grid, "pml_plain_parareal");
  check_same_grid(transfer.coarse, coarse.grid, "pml_plain_parareal");
  const size_t n = fine.grid.size(), N = n_couplings;
  const int K = std::max(iterations, 0);
  std::vector<double> err(size_t(std::max(K, 1)) * (N + 1)), states(4 * (N + 1) * n);
  int32_t div = 0;
  check(ptb_pml_parareal_run(fine.device_->h, coarse.device_->h, transfer_of(transfer), N, K, init.u.data(),
                             init.udot.data(), err.data(), nullptr, states.data(), &div));
  if (errors) {
    errors->assign(size_t(K), std::vector<double>(N + 1));
    for (int k = 0; k < K; ++k)
      std::copy(err.begin() + long(k) * long(N + 1), err.begin() + long(k + 1) * long(N + 1), (*errors)[size_t(k)].begin());
  }
  std::vector<PmlState> out;
  out.reserve(N + 1);
  for (size_t s = 0; s <= N; ++s) {
    auto field = [&](int f) {
      const auto b = states.begin() + long((size_t(f) * (N + 1) + s) * n);
      return std::vector<double>(b, b + long(n));
    };
    out.emplace_back(WaveState(fine.grid, field(0), field(1)), field(2), field(3));
  }
  return out;
}

}  // namespace paratime

