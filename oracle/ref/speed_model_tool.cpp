// ORACLE — test infrastructure only.  The reference's own speed-model text reader/writer
// (experiment.cpp:711-784, compiled verbatim into libparatime_ref.so) as a command-line filter,
// so tests compare against it in a separate process:
//   speed_model_tool write   stdin: "dim n0 n1 h0 h1" then n0*n1 values (%.17g) -> reference text
//   speed_model_tool read    stdin: speed-model text -> "dim n0 n1 h0 h1" then values (%.17g),
//                            or "CONFIG_ERROR <message>" (exit 5) / "ERROR <message>" (exit 4)
#include <cstdio>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "paratime/errors.hpp"
#include "paratime/experiment.hpp"
#include "paratime/grid.hpp"

using namespace paratime;

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "";
  try {
    if (mode == "write") {
      int dim = 0;
      std::size_t n0 = 0, n1 = 0;
      double h0 = 0, h1 = 0;
      std::cin >> dim >> n0 >> n1 >> h0 >> h1;
      const Grid g = dim == 1 ? Grid({n0}, {h0}) : Grid({n0, n1}, {h0, h1});
      std::vector<double> c(g.size());
      for (double& v : c) std::cin >> v;
      write_speed_model(SpeedField(g, c), std::cout);
      return 0;
    }
    if (mode == "read") {
      std::stringstream text;
      text << std::cin.rdbuf();
      const SpeedField f = read_speed_model(text);
      const Grid& g = f.grid;
      std::printf("%d %zu %zu %.17g %.17g\n", g.dim(), g.points(0), g.dim() == 2 ? g.points(1) : std::size_t(1),
                  g.spacing(0), g.dim() == 2 ? g.spacing(1) : 1.0);
      for (double v : f.c) std::printf("%.17g\n", v);
      return 0;
    }
  } catch (const ConfigError& e) {
    std::printf("CONFIG_ERROR %s\n", e.what());
    return 5;
  } catch (const std::exception& e) {
    std::printf("ERROR %s\n", e.what());
    return 4;
  }
  std::fprintf(stderr, "usage: speed_model_tool write|read\n");
  return 2;
}
