// ORACLE — test infrastructure only (tests/, bench.py cpu_baseline / --impl reference,
// smoke()).  Never linked into or called by the product library.
//
// Flat C entry points over the reference's own C++ API (compiled verbatim from
// /root/reference/proj/src by oracle/ref/Makefile) so Python tests can use the
// reference itself as the checker via ctypes.  Status codes:
//   0 ok, 1 std::invalid_argument, 2 PropagationDiverged, 3 std::domain_error,
//   4 other std::runtime_error / exception, 5 ConfigError.

#include <algorithm>
#include <chrono>
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "paratime/energy_map.hpp"
#include "paratime/errors.hpp"
#include "paratime/experiment.hpp"
#include "paratime/grid.hpp"
#include "paratime/parareal.hpp"
#include "paratime/procrustes.hpp"
#include "paratime/propagator.hpp"

using namespace paratime;

namespace {

thread_local std::string g_err;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 5;
  } catch (const PropagationDiverged& e) {
    g_err = e.what();
    return 2;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

Grid make_grid(int dim, std::size_t n0, std::size_t n1, double h0, double h1) {
  if (dim == 1) return Grid({n0}, {h0});
  return Grid({n0, n1}, {h0, h1});
}

std::vector<double> vec(const double* p, std::size_t n) { return std::vector<double>(p, p + n); }

GradientScheme scheme_of(int s) {
  switch (s) {
    case 0: return GradientScheme::fd2;
    case 1: return GradientScheme::fd4;
    case 2: return GradientScheme::fd6;
    case 3: return GradientScheme::fd8;
    case 4: return GradientScheme::spectral;
  }
  throw std::invalid_argument("bad scheme id");
}

// Static block partition over std::thread, identical to parareal.cpp:25-47.
template <typename Fn>
void static_parallel_for(std::size_t count, int workers, Fn&& fn) {
  if (count == 0) return;
  int hw = workers > 0 ? workers : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  const int n_threads = static_cast<int>(std::min<std::size_t>(static_cast<std::size_t>(hw), count));
  if (n_threads <= 1) {
    for (std::size_t i = 0; i < count; ++i) fn(i);
    return;
  }
  std::vector<std::thread> pool;
  const std::size_t chunk = (count + static_cast<std::size_t>(n_threads) - 1) / static_cast<std::size_t>(n_threads);
  for (int t = 0; t < n_threads; ++t) {
    const std::size_t lo = static_cast<std::size_t>(t) * chunk;
    const std::size_t hi = std::min(count, lo + chunk);
    if (lo >= hi) break;
    pool.emplace_back([lo, hi, &fn]() {
      for (std::size_t i = lo; i < hi; ++i) fn(i);
    });
  }
  for (auto& th : pool) th.join();
}

PhaseCorrector* as_corr(void* p) { return static_cast<PhaseCorrector*>(p); }

OMat mat(long rows, long cols, const double* colmajor) {
  OMat m(rows, cols);
  std::copy(colmajor, colmajor + rows * cols, m.data());
  return m;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }


int ref_laplacian(int dim, std::size_t n0, std::size_t n1, double h0, double h1, const double* f,
                  double* out) {
  return guarded([&] {
    const Grid g = make_grid(dim, n0, n1, h0, h1);
    const auto r = laplacian(vec(f, g.size()), g);
    std::copy(r.begin(), r.end(), out);
  });
}

int ref_cfl_check(int dim, std::size_t n0, std::size_t n1, double h0, double h1, const double* c,
                  double dt, std::size_t steps) {
  return guarded([&] {
    const Grid g = make_grid(dim, n0, n1, h0, h1);
    PropagatorConfig cfg(g, SpeedField(g, vec(c, g.size())), dt, steps);
    (void)cfg;
  });
}

// Batched propagate_coupling (propagator.cpp:95-105) over `batch` slice-major states,
// in place; slices run on `workers` std::threads with parareal.cpp's partition.
// diverged[b] = 1 where the reference threw PropagationDiverged (state then untouched).
int ref_propagate(int dim, std::size_t n0, std::size_t n1, double h0, double h1, const double* c,
                  double dt, std::size_t steps, std::size_t batch, double* u, double* udot,
                  int workers, int* diverged) {
  return guarded([&] {
    const Grid g = make_grid(dim, n0, n1, h0, h1);
    const std::size_t n = g.size();
    const PropagatorConfig cfg(g, SpeedField(g, vec(c, n)), dt, steps);
    static_parallel_for(batch, workers, [&](std::size_t b) {
      const WaveState in(g, vec(u + b * n, n), vec(udot + b * n, n));
      try {
        const WaveState out = propagate_coupling(in, cfg);
        std::copy(out.u.begin(), out.u.end(), u + b * n);
        std::copy(out.udot.begin(), out.udot.end(), udot + b * n);
        if (diverged) diverged[b] = 0;
      } catch (const PropagationDiverged&) {
        if (diverged) diverged[b] = 1;
      }
    });
  });
}

int ref_step(int dim, std::size_t n0, std::size_t n1, double h0, double h1, const double* c,
             double dt, double* u, double* udot) {
  return guarded([&] {
    const Grid g = make_grid(dim, n0, n1, h0, h1);
    const std::size_t n = g.size();
    const PropagatorConfig cfg(g, SpeedField(g, vec(c, n)), dt, 1);
    const WaveState out = step(WaveState(g, vec(u, n), vec(udot, n)), cfg);
    std::copy(out.u.begin(), out.u.end(), u);
    std::copy(out.udot.begin(), out.udot.end(), udot);
  });
}

int ref_restrict(int dim, std::size_t c0, std::size_t c1, double ch0, double ch1, std::size_t f0,
                 std::size_t f1, double fh0, double fh1, const double* fine, double* coarse) {
  return guarded([&] {
    const GridTransfer t(make_grid(dim, c0, c1, ch0, ch1), make_grid(dim, f0, f1, fh0, fh1),
                         InterpKind::linear);
    const auto r = restrict_field(vec(fine, t.fine.size()), t);
    std::copy(r.begin(), r.end(), coarse);
  });
}

int ref_interpolate(int dim, std::size_t c0, std::size_t c1, double ch0, double ch1, std::size_t f0,
                    std::size_t f1, double fh0, double fh1, int kind, const double* coarse,
                    double* fine) {
  return guarded([&] {
    const GridTransfer t(make_grid(dim, c0, c1, ch0, ch1), make_grid(dim, f0, f1, fh0, fh1),
                         kind == 0 ? InterpKind::fourier : InterpKind::linear);
    const auto r = interpolate_field(vec(coarse, t.coarse.size()), t);
    std::copy(r.begin(), r.end(), fine);
  });
}

int ref_gradient_axis(int dim, std::size_t n0, std::size_t n1, double h0, double h1,
                      const double* f, int axis, int scheme, double* out) {
  return guarded([&] {
    const Grid g = make_grid(dim, n0, n1, h0, h1);
    const auto r = gradient_axis(vec(f, g.size()), g, axis, scheme_of(scheme));
    std::copy(r.begin(), r.end(), out);
  });
}

// stacked layout = stack_components (procrustes.cpp:129-142): [grad axis0; ...; momentum]
int ref_energy_components(int dim, std::size_t n0, std::size_t n1, double h0, double h1,
                          const double* c, int scheme, const double* u, const double* udot,
                          double* stacked, double* mean_u) {
  return guarded([&] {
    const Grid g = make_grid(dim, n0, n1, h0, h1);
    const std::size_t n = g.size();
    const EnergyComponents comp = to_energy_components(WaveState(g, vec(u, n), vec(udot, n)),
                                                       SpeedField(g, vec(c, n)), scheme_of(scheme));
    const auto s = stack_components(comp);
    std::copy(s.begin(), s.end(), stacked);
    *mean_u = comp.mean_u;
  });
}

int ref_from_energy_components(int dim, std::size_t n0, std::size_t n1, double h0, double h1,
                               const double* c, const double* stacked, double mean_u, double* u,
                               double* udot) {
  return guarded([&] {
    const Grid g = make_grid(dim, n0, n1, h0, h1);
    const std::size_t n = g.size();
    const EnergyComponents comp =
        unstack_components(vec(stacked, (static_cast<std::size_t>(g.dim()) + 1) * n), g, mean_u);
    const WaveState s = from_energy_components(comp, SpeedField(g, vec(c, n)));
    std::copy(s.u.begin(), s.u.end(), u);
    std::copy(s.udot.begin(), s.udot.end(), udot);
  });
}

int ref_energy(int dim, std::size_t n0, std::size_t n1, double h0, double h1, const double* c,
               int scheme, const double* u, const double* udot, double* out) {
  return guarded([&] {
    const Grid g = make_grid(dim, n0, n1, h0, h1);
    const std::size_t n = g.size();
    *out = energy(WaveState(g, vec(u, n), vec(udot, n)), SpeedField(g, vec(c, n)), scheme_of(scheme));
  });
}

int ref_energy_error(int dim, std::size_t n0, std::size_t n1, double h0, double h1,
                     const double* c, int scheme, const double* ua, const double* udota,
                     const double* ub, const double* udotb, double* out) {
  return guarded([&] {
    const Grid g = make_grid(dim, n0, n1, h0, h1);
    const std::size_t n = g.size();
    *out = energy_error(WaveState(g, vec(ua, n), vec(udota, n)), WaveState(g, vec(ub, n), vec(udotb, n)),
                        SpeedField(g, vec(c, n)), scheme_of(scheme));
  });
}

int ref_l2_error(int dim, std::size_t n0, std::size_t n1, double h0, double h1, const double* ua,
                 const double* ub, double* out) {
  return guarded([&] {
    const Grid g = make_grid(dim, n0, n1, h0, h1);
    const std::size_t n = g.size();
    const std::vector<double> z(n, 0.0);
    *out = l2_error(WaveState(g, vec(ua, n), z), WaveState(g, vec(ub, n), z));
  });
}

// ---- Procrustes (restated on LAPACK, procrustes_lapack.cpp) --------------------------

void ref_corrector_free(void* p) { delete as_corr(p); }

int ref_procrustes_solve(long rows, long cols, const double* F, const double* G, double tol,
                         void** out) {
  return guarded([&] {
    *out = new PhaseCorrector(procrustes_solve(mat(rows, cols, F), mat(rows, cols, G), tol));
  });
}

int ref_update_svd(void* corr, long rows, long cols, const double* F, const double* G, double tol,
                   void** out) {
  return guarded([&] {
    const PhaseCorrector empty;
    const PhaseCorrector& c = corr ? *as_corr(corr) : empty;
    *out = new PhaseCorrector(update_svd(c, mat(rows, cols, F), mat(rows, cols, G), tol));
  });
}

int ref_corrector_shape(void* corr, long* rows, long* rank) {
  return guarded([&] {
    *rows = as_corr(corr)->rows();
    *rank = as_corr(corr)->rank();
  });
}

int ref_corrector_factors(void* corr, double* X, double* sv, double* Y) {
  return guarded([&] {
    const PhaseCorrector& c = *as_corr(corr);
    const long n = c.rows() * c.rank();
    std::copy(c.left().data(), c.left().data() + n, X);
    std::copy(c.right().data(), c.right().data() + n, Y);
    std::copy(c.singular_values().begin(), c.singular_values().end(), sv);
  });
}

int ref_corrector_drop_leading(void* corr, long count, void** out) {
  return guarded([&] { *out = new PhaseCorrector(as_corr(corr)->drop_leading(count)); });
}

int ref_corrector_apply(void* corr, const double* v, double* out) {
  return guarded([&] {
    const PhaseCorrector& c = *as_corr(corr);
    const auto r = c.apply(vec(v, static_cast<std::size_t>(c.rows())));
    std::copy(r.begin(), r.end(), out);
  });
}

int ref_relative_residual(void* corr, long rows, long cols, const double* F, const double* G,
                          double* out) {
  return guarded([&] {
    *out = relative_residual(*as_corr(corr), mat(rows, cols, F), mat(rows, cols, G));
  });
}

// ---- drivers (parareal.cpp verbatim) ---------------------------------------------------

struct RefRunSpec {
  int dim;
  std::size_t fine_n[2];
  double fine_h[2];
  std::size_t coarse_n[2];
  double coarse_h[2];
  double dt_fine;
  std::size_t m_fine;
  double dt_coarse;
  std::size_t m_coarse;
  double T;
  double dt_com;
  std::size_t n_couplings;
  int interp;          // 0 fourier, 1 linear
  int iterations;
  int variant;         // 0 plain, 1 theta, 2 corrected_coarse_only, 3 omega_identity
  int scheme;          // data-matrix gradient
  int metric_scheme;   // error seminorm
  double tol;
  int remove_leading;
  int workers;
};

// Outputs (caller-allocated, K = iterations, N = n_couplings):
//   energy_err, l2_err : (K+1)*(N+1) row-major [k][n]
//   residual, rank, diverged : K+1
//   states (nullable): (K+1)*(N+1)*2*Nf — [k][n][u|udot][pt]
//   reference (nullable): (N+1)*2*Nf
//   phase_ms (nullable): 1 value, wall ms of the driver call
int ref_parareal_run(const RefRunSpec* s, const double* c_fine, const double* c_coarse,
                     const double* u0, const double* udot0, double* energy_err, double* l2_err,
                     double* residual, int* rank, int* diverged, double* states, double* reference,
                     double* wall_ms) {
  return guarded([&] {
    const Grid fg = make_grid(s->dim, s->fine_n[0], s->fine_n[1], s->fine_h[0], s->fine_h[1]);
    const Grid cg = make_grid(s->dim, s->coarse_n[0], s->coarse_n[1], s->coarse_h[0], s->coarse_h[1]);
    const std::size_t nf = fg.size(), nc = cg.size();
    PropagatorConfig fine_cfg(fg, SpeedField(fg, vec(c_fine, nf)), s->dt_fine, s->m_fine);
    PropagatorConfig coarse_cfg(cg, SpeedField(cg, vec(c_coarse, nc)), s->dt_coarse, s->m_coarse);
    const CouplingSchedule schedule(s->T, s->dt_com, s->n_couplings, fine_cfg, coarse_cfg);
    const GridTransfer transfer(cg, fg, s->interp == 0 ? InterpKind::fourier : InterpKind::linear);
    const WaveState init(fg, vec(u0, nf), vec(udot0, nf));
    DriverOptions driver;
    driver.metric_scheme = scheme_of(s->metric_scheme);
    driver.workers = s->workers;
    driver.keep_states = states != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    ParaRun run;
    if (s->variant == 0) {
      run = plain_parareal(init, schedule, transfer, s->iterations, driver);
    } else {
      ThetaOptions opts;
      opts.scheme = scheme_of(s->scheme);
      opts.tol = s->tol;
      opts.omega_identity = s->variant == 3;
      opts.remove_leading = s->remove_leading;
      opts.driver = driver;
      run = s->variant == 2 ? corrected_coarse_only(init, schedule, transfer, s->iterations, opts)
                            : theta_parareal(init, schedule, transfer, s->iterations, opts);
    }
    if (wall_ms)
      *wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    const std::size_t N = s->n_couplings;
    for (std::size_t k = 0; k < run.iterations.size(); ++k) {
      const IterationRecord& rec = run.iterations[k];
      for (std::size_t n = 0; n <= N; ++n) {
        energy_err[k * (N + 1) + n] = rec.energy_err[n];
        l2_err[k * (N + 1) + n] = rec.l2_err[n];
      }
      residual[k] = rec.residual;
      rank[k] = rec.rank;
      diverged[k] = rec.diverged ? 1 : 0;
      if (states)
        for (std::size_t n = 0; n <= N; ++n) {
          double* dst = states + ((k * (N + 1) + n) * 2) * nf;
          std::copy(rec.states[n].u.begin(), rec.states[n].u.end(), dst);
          std::copy(rec.states[n].udot.begin(), rec.states[n].udot.end(), dst + nf);
        }
    }
    if (reference)
      for (std::size_t n = 0; n <= N; ++n) {
        double* dst = reference + n * 2 * nf;
        std::copy(run.reference[n].u.begin(), run.reference[n].u.end(), dst);
        std::copy(run.reference[n].udot.begin(), run.reference[n].udot.end(), dst + nf);
      }
  });
}

// Resolve a preset (experiment.cpp:225-375) or config text plus "key=value" overrides
// (newline separated) into a RefRunSpec and its arrays (experiment.cpp:503-557).
// Call once with arrays null to get sizes (spec filled), then again with arrays.
int ref_build_setup(const char* preset_name, const char* config_text, const char* overrides,
                    RefRunSpec* spec, double* c_fine, double* c_coarse, double* u0, double* udot0) {
  return guarded([&] {
    ExperimentConfig cfg;
    if (preset_name && *preset_name) {
      cfg = preset(preset_name);
    } else {
      std::istringstream is(config_text ? config_text : "");
      cfg = parse_config(is);
    }
    if (overrides) {
      std::istringstream os(overrides);
      std::string line;
      while (std::getline(os, line)) {
        const auto eq = line.find('=');
        if (eq == std::string::npos) continue;
        apply_override(cfg, line.substr(0, eq), line.substr(eq + 1));
      }
    }
    const ExperimentSetup st = build_setup(cfg);
    spec->dim = st.fine_grid.dim();
    for (int a = 0; a < 2; ++a) {
      const bool has = a < spec->dim;
      spec->fine_n[a] = has ? st.fine_grid.points(a) : 1;
      spec->fine_h[a] = has ? st.fine_grid.spacing(a) : 1.0;
      spec->coarse_n[a] = has ? st.coarse_grid.points(a) : 1;
      spec->coarse_h[a] = has ? st.coarse_grid.spacing(a) : 1.0;
    }
    spec->dt_fine = st.schedule.fine_cfg.dt;
    spec->m_fine = st.schedule.fine_cfg.steps_per_coupling;
    spec->dt_coarse = st.schedule.coarse_cfg.dt;
    spec->m_coarse = st.schedule.coarse_cfg.steps_per_coupling;
    spec->T = st.schedule.T;
    spec->dt_com = st.schedule.dt_com;
    spec->n_couplings = st.schedule.n_couplings;
    spec->interp = st.transfer.kind == InterpKind::fourier ? 0 : 1;
    spec->iterations = cfg.iterations;
    spec->variant = cfg.variant == Variant::plain ? 0
                    : cfg.variant == Variant::theta ? 1
                    : cfg.variant == Variant::corrected_coarse_only ? 2 : 3;
    spec->scheme = static_cast<int>(cfg.gradient);
    spec->metric_scheme = static_cast<int>(cfg.gradient);
    spec->tol = cfg.tol;
    spec->remove_leading = cfg.remove_count;
    spec->workers = cfg.workers;
    if (c_fine) std::copy(st.fine_speed.c.begin(), st.fine_speed.c.end(), c_fine);
    if (c_coarse) std::copy(st.coarse_speed.c.begin(), st.coarse_speed.c.end(), c_coarse);
    if (u0) std::copy(st.init.u.begin(), st.init.u.end(), u0);
    if (udot0) std::copy(st.init.udot.begin(), st.init.udot.end(), udot0);
  });
}

}  // extern "C"
