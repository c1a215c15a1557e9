// Host-side text formats of the drop-in API — the data formats on either side of the hot path.
//
//   corrector checkpoint   PhaseCorrector::save / load        (reference procrustes.cpp:95-127)
//   speed-model text        read / ingest / write_speed_model  (experiment.hpp:84-90)
//   run-record CSVs         errors.csv / residuals.csv / summary.csv (experiment.cpp:596-628)
//   bilinear resampling     bilinear_resample                  (grid.cpp:252-298)
//
// The byte layout (headers, separators, "%.17g" numbers) and the exception types/messages are
// the contract and match the reference; the code is organised around three small helpers of
// this build: a token reader with typed failures, a line builder that formats numbers once,
// and per-axis resampling taps.

#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <istream>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "paratime/errors.hpp"
#include "paratime/grid.hpp"
#include "paratime/procrustes.hpp"
#include "paratime/run_files.hpp"
#include "paratime/speed_model.hpp"
#include "paratime_b200.h"

namespace paratime {
namespace {

// -------------------------------------------------------------- helpers

// Pulls whitespace-separated values with stream-extraction semantics; every failure throws E
// with the caller's message.
template <typename E>
class TokenReader {
 public:
  explicit TokenReader(std::istream& is) : is_(is) {}
  template <typename T>
  T get(const char* what) {
    T v{};
    if (!(is_ >> v)) throw E(what);
    return v;
  }
  template <typename T>
  void fill(T* dst, std::size_t count, const char* what) {
    for (std::size_t i = 0; i < count; ++i) dst[i] = get<T>(what);
  }
  bool exhausted() {
    double extra;
    return !(is_ >> extra);
  }

 private:
  std::istream& is_;
};

// One output line: cells joined by `sep`, doubles as "%.17g" (the reference's fmt(),
// experiment.cpp:19-23; iostream precision 17 prints the same digits).
class Line {
 public:
  explicit Line(char sep) : sep_(sep) {}
  Line& num(double v) {
    char b[40];
    const int k = std::snprintf(b, sizeof b, "%.17g", v);
    return cell(b, std::size_t(k));
  }
  Line& num(long long v) { return text(std::to_string(v)); }
  Line& num(std::size_t v) { return text(std::to_string(v)); }
  Line& num(int v) { return text(std::to_string(v)); }
  Line& text(const std::string& s) { return cell(s.data(), s.size()); }
  void emit(std::ostream& os) { os << buf_ << '\n'; }

 private:
  Line& cell(const char* p, std::size_t n) {
    if (!first_) buf_.push_back(sep_);
    first_ = false;
    buf_.append(p, n);
    return *this;
  }
  std::string buf_;
  char sep_;
  bool first_ = true;
};

void emit_rows(std::ostream& os, const double* a, std::size_t rows, std::size_t cols, bool row_major) {
  for (std::size_t i = 0; i < rows; ++i) {
    Line l(' ');
    for (std::size_t j = 0; j < cols; ++j) l.num(row_major ? a[i * cols + j] : a[j * rows + i]);
    l.emit(os);
  }
}

// bilinear taps along one axis: destination j samples source position j * src/dst (grid.cpp:252-260)
struct Tap {
  std::size_t lo, hi;
  double w;
};
std::vector<Tap> axis_taps(std::size_t src, std::size_t dst) {
  std::vector<Tap> t(dst);
  const double scale = static_cast<double>(src) / static_cast<double>(dst);
  for (std::size_t j = 0; j < dst; ++j) {
    const double pos = static_cast<double>(j) * scale, base = std::floor(pos);
    t[j].lo = static_cast<std::size_t>(base) % src;
    t[j].hi = (t[j].lo + 1) % src;
    t[j].w = pos - base;
  }
  return t;
}

// speed-model table: "ny nx dy dx" then ny*nx positive finite values (experiment.hpp:84-90)
struct SpeedTable {
  std::size_t ny = 0, nx = 0;
  double dy = 0.0, dx = 0.0;
  std::vector<double> c;
};

SpeedTable read_table(std::istream& is) {
  TokenReader<ConfigError> in(is);
  static const char* kHeader = "speed model: bad header (want: ny nx dy dx)";
  const long ny = in.get<long>(kHeader), nx = in.get<long>(kHeader);
  SpeedTable t;
  t.dy = in.get<double>(kHeader);
  t.dx = in.get<double>(kHeader);
  if (ny < 1 || nx < 1) throw ConfigError("speed model: nonpositive shape");
  if (!(t.dx > 0.0) || (ny > 1 && !(t.dy > 0.0))) throw ConfigError("speed model: nonpositive spacing");
  t.ny = static_cast<std::size_t>(ny);
  t.nx = static_cast<std::size_t>(nx);
  t.c.resize(t.ny * t.nx);
  for (double& v : t.c) {
    v = in.get<double>("speed model: truncated value table");
    if (!(v > 0.0) || !std::isfinite(v)) throw ConfigError("speed model: wave speed entries must be positive and finite");
  }
  if (!in.exhausted()) throw ConfigError("speed model: trailing values beyond ny*nx");
  return t;
}

SpeedField table_field(SpeedTable t) {
  if (t.nx < 4 || (t.ny > 1 && t.ny < 4))
    throw ConfigError("speed model: too few points for a grid; resample to a target size");
  Grid g = t.ny == 1 ? Grid({t.nx}, {t.dx}) : Grid({t.ny, t.nx}, {t.dy, t.dx});
  return SpeedField(std::move(g), std::move(t.c));
}

std::ifstream open_model(const std::string& path) {
  std::ifstream is(path);
  if (!is) throw ConfigError("cannot open speed model: " + path);
  return is;
}

}  // namespace

// C-string hand-off of the C ABI: `needed` = bytes incl. the terminator; copied when it fits
void copy_out(const std::string& text, char* buf, std::size_t len, std::size_t* needed) {
  *needed = text.size() + 1;
  if (buf && len >= text.size() + 1) std::memcpy(buf, text.c_str(), text.size() + 1);
}

// -------------------------------------------------------------- bilinear resampling (grid.hpp)

std::vector<double> bilinear_resample(const std::vector<double>& src, std::size_t sny, std::size_t snx,
                                      std::size_t dny, std::size_t dnx) {
  if (src.size() != sny * snx) throw std::invalid_argument("bilinear_resample: field size does not match source shape");
  if (!sny || !snx || !dny || !dnx) throw std::invalid_argument("bilinear_resample: empty shape");
  const std::vector<Tap> ty = axis_taps(sny, dny), tx = axis_taps(snx, dnx);
  std::vector<double> out(dny * dnx);
  double* o = out.data();
  for (const Tap& y : ty) {
    const double* r0 = src.data() + y.lo * snx;
    const double* r1 = src.data() + y.hi * snx;
    for (const Tap& x : tx)  // rows blended first, then the two rows (grid.cpp:278-282 order)
      *o++ = (1.0 - y.w) * ((1.0 - x.w) * r0[x.lo] + x.w * r0[x.hi]) + y.w * ((1.0 - x.w) * r1[x.lo] + x.w * r1[x.hi]);
  }
  return out;
}

std::vector<double> bilinear_resample(const std::vector<double>& src, const Grid& sg, const Grid& dg) {
  if (src.size() != sg.size()) throw std::invalid_argument("bilinear_resample: field size does not match source grid");
  if (sg.dim() != dg.dim()) throw std::invalid_argument("bilinear_resample: dimension mismatch");
  const auto rows = [](const Grid& g) { return g.dim() == 1 ? std::size_t(1) : g.points(0); };
  const auto cols = [](const Grid& g) { return g.points(g.dim() - 1); };
  return bilinear_resample(src, rows(sg), cols(sg), rows(dg), cols(dg));
}

// -------------------------------------------------------------- corrector checkpoint (procrustes.hpp)

void PhaseCorrector::save(std::ostream& os) const {
  Line head(' ');
  head.num(static_cast<long long>(rows())).num(static_cast<long long>(rank())).emit(os);
  const std::size_t m = static_cast<std::size_t>(rows()), r = static_cast<std::size_t>(rank());
  emit_rows(os, left_.data(), m, r, false);  // column-major factor, printed row by row
  emit_rows(os, sv_.data(), 1, r, true);
  emit_rows(os, right_.data(), m, r, false);
}

PhaseCorrector PhaseCorrector::load(std::istream& is) {
  TokenReader<std::runtime_error> in(is);
  const Index m = in.get<Index>("corrector checkpoint: bad header");
  const Index r = in.get<Index>("corrector checkpoint: bad header");
  if (m < 0 || r < 0) throw std::runtime_error("corrector checkpoint: bad header");
  const auto factor = [&in, m, r] {
    Matrix f(m, r);
    for (Index i = 0; i < m; ++i)  // the file is row by row; the matrix is column-major
      for (Index j = 0; j < r; ++j) f(i, j) = in.get<double>("corrector checkpoint: truncated matrix block");
    return f;
  };
  Matrix X = factor();
  std::vector<double> sv(static_cast<std::size_t>(r));
  in.fill(sv.data(), sv.size(), "corrector checkpoint: truncated values");
  Matrix Y = factor();
  return PhaseCorrector(std::move(X), std::move(sv), std::move(Y), 0.0);
}

// -------------------------------------------------------------- speed model (speed_model.hpp)

SpeedField read_speed_model(std::istream& is) { return table_field(read_table(is)); }

SpeedField ingest_speed_model(const std::string& path) {
  std::ifstream is = open_model(path);
  return read_speed_model(is);
}

SpeedField ingest_speed_model(const std::string& path, const Grid& target) {
  std::ifstream is = open_model(path);
  SpeedTable t = read_table(is);
  if (target.dim() == 2 && t.ny == 1) throw ConfigError("speed model: 1D file cannot fill a 2D grid");
  const std::size_t ty = target.dim() == 1 ? 1 : target.points(0);
  return SpeedField(target, bilinear_resample(t.c, t.ny, t.nx, ty, target.points(target.dim() - 1)));
}

void write_speed_model(const SpeedField& field, std::ostream& os) {
  const Grid& g = field.grid;
  const bool two = g.dim() == 2;
  const std::size_t ny = two ? g.points(0) : 1, nx = g.points(g.dim() - 1);
  Line head(' ');
  head.num(ny).num(nx).num(two ? g.spacing(0) : 1.0).num(g.spacing(g.dim() - 1)).emit(os);
  emit_rows(os, field.c.data(), ny, nx, true);
}

// -------------------------------------------------------------- run-record CSVs (run_files.hpp)

void write_errors_csv(const ParaRun& run, std::ostream& os) {
  os << "iteration,coupling,energy_error,l2_error,diverged\n";
  for (std::size_t k = 0; k < run.iterations.size(); ++k) {
    const IterationRecord& it = run.iterations[k];
    for (std::size_t n = 0; n < it.energy_err.size(); ++n)
      Line(',').num(k).num(n).num(it.energy_err[n]).num(it.l2_err[n]).num(int(it.diverged)).emit(os);
  }
}

void write_residuals_csv(const ParaRun& run, bool plain, std::ostream& os) {
  os << "iteration,residual,rank\n";
  if (plain) return;  // plain parareal has no corrector: header only
  for (std::size_t k = 1; k < run.iterations.size(); ++k)
    Line(',').num(k).num(run.iterations[k].residual).num(int(run.iterations[k].rank)).emit(os);
}

void write_summary_csv(const ParaRun& run, std::ostream& os) {
  os << "iteration,energy_error,l2_error,diverged\n";
  for (std::size_t k = 0; k < run.iterations.size(); ++k) {
    const IterationRecord& it = run.iterations[k];
    Line(',').num(k).num(it.energy_err.back()).num(it.l2_err.back()).num(int(it.diverged)).emit(os);
  }
}

void write_run_csv(const ParaRun& run, bool plain, const std::string& dir) {
  namespace fs = std::filesystem;
  fs::create_directories(dir);
  std::ofstream errors(fs::path(dir) / "errors.csv"), residuals(fs::path(dir) / "residuals.csv"),
      summary(fs::path(dir) / "summary.csv");
  write_errors_csv(run, errors);
  write_residuals_csv(run, plain, residuals);
  write_summary_csv(run, summary);
}

}  // namespace paratime

// -------------------------------------------------------------- C ABI (paratime_b200.h)

namespace ptb {
extern thread_local std::string g_last_error;  // capi.cpp (ptb_last_error)
}

namespace {
// ConfigError -> PTB_CONFIG, std::invalid_argument -> PTB_INVALID_ARGUMENT
template <typename Fn>
ptb_status host_guarded(Fn&& fn) {
  try {
    fn();
    return PTB_OK;
  } catch (const paratime::ConfigError& e) {
    ptb::g_last_error = e.what();
    return PTB_CONFIG;
  } catch (const std::invalid_argument& e) {
    ptb::g_last_error = e.what();
    return PTB_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    ptb::g_last_error = e.what();
    return PTB_UNSUPPORTED;
  }
}
}  // namespace

extern "C" ptb_status ptb_speed_model_write(const ptb_grid* grid, const double* c, char* buf, size_t len,
                                            size_t* needed) {
  return host_guarded([&] {
    if (!grid || !c || !needed) throw std::invalid_argument("speed_model_write: null argument");
    const paratime::Grid g(std::vector<std::size_t>(grid->n, grid->n + grid->dim),
                           std::vector<double>(grid->h, grid->h + grid->dim));
    std::ostringstream os;
    paratime::write_speed_model(paratime::SpeedField(g, std::vector<double>(c, c + g.size())), os);
    paratime::copy_out(os.str(), buf, len, needed);
  });
}

extern "C" ptb_status ptb_speed_model_read(const char* text, ptb_grid* grid, double* c, size_t cap,
                                           size_t* npoints) {
  return host_guarded([&] {
    if (!text || !grid || !npoints) throw std::invalid_argument("speed_model_read: null argument");
    std::istringstream is(text);
    const paratime::SpeedField f = paratime::read_speed_model(is);
    grid->dim = f.grid.dim();
    for (int a = 0; a < 2; ++a) {
      grid->n[a] = a < f.grid.dim() ? f.grid.points(a) : 0;
      grid->h[a] = a < f.grid.dim() ? f.grid.spacing(a) : 0.0;
    }
    *npoints = f.c.size();
    if (c && cap >= f.c.size()) std::copy(f.c.begin(), f.c.end(), c);
  });
}

// run-record CSV text of K iterations x (N + 1) couplings given as row-major arrays;
// which: 0 errors.csv, 1 residuals.csv, 2 summary.csv
extern "C" ptb_status ptb_run_csv(size_t iterations, size_t couplings, const double* energy_err, const double* l2_err,
                                  const double* residual, const int* rank, const int* diverged, int plain, int which,
                                  char* buf, size_t len, size_t* needed) {
  return host_guarded([&] {
    if (!energy_err || !l2_err || !residual || !rank || !diverged || !needed)
      throw std::invalid_argument("run_csv: null argument");
    if (which < 0 || which > 2) throw std::invalid_argument("run_csv: which must be 0, 1 or 2");
    paratime::ParaRun run;
    run.iterations.resize(iterations);
    for (size_t k = 0; k < iterations; ++k) {
      paratime::IterationRecord& rec = run.iterations[k];
      rec.energy_err.assign(energy_err + k * couplings, energy_err + (k + 1) * couplings);
      rec.l2_err.assign(l2_err + k * couplings, l2_err + (k + 1) * couplings);
      rec.residual = residual[k];
      rec.rank = rank[k];
      rec.diverged = diverged[k] != 0;
    }
    std::ostringstream os;
    if (which == 0) paratime::write_errors_csv(run, os);
    else if (which == 1) paratime::write_residuals_csv(run, plain != 0, os);
    else paratime::write_summary_csv(run, os);
    paratime::copy_out(os.str(), buf, len, needed);
  });
}
