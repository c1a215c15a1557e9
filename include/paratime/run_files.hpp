// paratime_b200: the run-record CSV schemas of the reference's experiment harness
// (/root/reference/proj/src/experiment.cpp:596-628, write_run_files): errors.csv, residuals.csv and
// summary.csv of a ParaRun, byte-equal to the reference's writer (numbers as "%.17g",
// experiment.cpp:19-23).  config.txt and meta.txt describe the harness configuration and are
// out of scope with it.
#pragma once

#include <iosfwd>
#include <string>

#include "paratime/parareal.hpp"

namespace paratime {

/// "iteration,coupling,energy_error,l2_error,diverged", one row per (k, n)
void write_errors_csv(const ParaRun& run, std::ostream& os);
/// "iteration,residual,rank", one row per k >= 1; header only for plain parareal
void write_residuals_csv(const ParaRun& run, bool plain, std::ostream& os);
/// "iteration,energy_error,l2_error,diverged": the last coupling of every iteration
void write_summary_csv(const ParaRun& run, std::ostream& os);
/// the three files into `dir` (created if missing)
void write_run_csv(const ParaRun& run, bool plain, const std::string& dir);

}  // namespace paratime
