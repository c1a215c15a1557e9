// ORACLE — test infrastructure only.  The reference's own harness entry run_experiment
// (experiment.cpp:631-668, compiled verbatim into libparatime_ref.so) as a command-line tool, so the
// run-record CSVs (errors.csv, residuals.csv, summary.csv: write_run_files, experiment.cpp:596-628)
// come from the reference itself (in a separate process: its ofstream/filesystem use does not mix
// with the Python process):
//   run_experiment_tool <preset> <out_dir> [key=value ...]
#include <iostream>
#include <string>

#include "paratime/errors.hpp"
#include "paratime/experiment.hpp"

using namespace paratime;

int main(int argc, char** argv) {
  if (argc < 3) {
    std::cerr << "usage: run_experiment_tool <preset> <out_dir> [key=value ...]\n";
    return 2;
  }
  try {
    ExperimentConfig cfg = preset(argv[1]);
    for (int i = 3; i < argc; ++i) {
      const std::string kv = argv[i];
      const auto eq = kv.find('=');
      if (eq == std::string::npos) continue;
      apply_override(cfg, kv.substr(0, eq), kv.substr(eq + 1));
    }
    cfg.out = argv[2];
    return run_experiment(cfg);
  } catch (const std::exception& e) {
    std::cerr << "ERROR " << e.what() << "\n";
    return 4;
  }
}
